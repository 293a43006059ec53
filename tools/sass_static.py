"""Static opcode mix of one kernel's hottest loop, from cuobjdump (no GPU needed).

usage: python tools/sass_static.py 'acoustic3d_vecq_kernel<8, true, 4>' [lib.so]

Finds the backward branch spanning the most instructions that is not itself
inside... (simply: the longest backward-branch span) and counts opcodes inside
it. For the stencil kernels that span is the plane loop (one or two steps per
pass), so the counts are per thread per pass.
"""
import collections
import re
import subprocess
import sys


def kernel_sass(lib, want):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    blocks = out.split("\t\tFunction : ")
    for b in blocks[1:]:
        name = b.split("\n", 1)[0].strip()
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        if want in dem.replace("sfb::", ""):
            return dem, b
    raise SystemExit(f"kernel {want!r} not found")


def main():
    want = sys.argv[1]
    lib = sys.argv[2] if len(sys.argv) > 2 else "paper_1609_03361_b200/libsf_b200.so"
    dem, body = kernel_sass(lib, want)
    ins = []  # (addr, opcode, text)
    for line in body.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if not m:
            continue
        addr = int(m.group(1), 16)
        text = m.group(2).strip()
        toks = [t for t in text.split() if not t.startswith("@")]
        ins.append((addr, toks[0] if toks else "?", text))
    # longest backward branch
    best = (0, 0, 0)
    for addr, op, text in ins:
        if op.startswith("BRA"):
            m = re.search(r"0x([0-9a-f]+)", text)
            if m:
                tgt = int(m.group(1), 16)
                if tgt < addr and addr - tgt > best[0]:
                    best = (addr - tgt, tgt, addr)
    _, lo, hi = best
    cnt = collections.Counter()
    for addr, op, text in ins:
        if lo <= addr <= hi:
            cnt[op.split(".")[0] if not op.startswith(("LDS", "STG", "LDG", "IMAD")) else
                ".".join(op.split(".")[:2])] += 1
    total = sum(cnt.values())
    print(f"{dem}: {len(ins)} instructions, hottest loop {total} "
          f"(0x{lo:x}..0x{hi:x})")
    print("  " + ", ".join(f"{k} {v}" for k, v in cnt.most_common(30)))


if __name__ == "__main__":
    main()
