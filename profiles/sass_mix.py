"""Per-opcode instruction mix of one ncu source-page export (SASS view).
usage: python profiles/sass_mix.py gpurun_out/prof/vec_c2.sass.csv POINTS TITLE"""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si, ei = h.index("Source"), h.index("Instructions Executed")
pts = float(sys.argv[2])
by_op = collections.Counter()
total = 0
for r in rows[2:]:
    if len(r) <= ei:
        continue
    n = int(r[ei] or 0)
    src = r[si].strip()
    toks = [t for t in src.replace(";", "").split() if not t.startswith("@")]
    if not toks:
        continue
    by_op[toks[0].split(".")[0]] += n
    total += n
print(f"# SASS instruction mix of {sys.argv[3]}")
print("# ncu --set full --import-source on, source page (Instructions Executed per SASS line)")
print(f"total warp-instructions {total}; thread-instructions per interior point {32 * total / pts:.1f}")
print("per point by opcode: " + ", ".join(f"{op} {32 * n / pts:.1f}" for op, n in by_op.most_common(22)))
