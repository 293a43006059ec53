"""Round-2 ncu summaries: one block per `--set full` capture exported by
tools/ncu_one.sh (gpurun_out/prof/<name>.raw.csv), with the pipe and memory
lenses the verdict asked for (FMA pipe, shared-memory wavefronts, L2 sectors,
DRAM bytes vs the algorithmic bytes).

    python profiles/summarize_r2.py name:points:alg_bytes_per_point [...]
"""
import csv
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors.sum", "lts__t_sectors.sum.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "inst_executed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def block(name, pts, alg):
    rr = list(csv.reader(open(f"gpurun_out/prof/{name}.raw.csv")))
    d, u = dict(zip(rr[0], rr[2])), dict(zip(rr[0], rr[1]))
    out = [f"## {name}"]
    for k in KEYS:
        if k in d:
            out.append(f"{k} = {d[k]} {u.get(k, '')}".rstrip())
    dram = sum(float(d[k]) * SCALE[u[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    out.append(f"DRAM bytes per launch = {dram / 1e6:.1f} MB; algorithmic {alg} B/pt x {pts} pts "
               f"= {alg * pts / 1e6:.1f} MB ({dram / (alg * pts):.3f}x)")
    if "lts__t_sectors.sum" in d:
        out.append(f"L2 bytes per point = {32 * float(d['lts__t_sectors.sum']) / pts:.2f}")
    if "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum" in d:
        out.append("shared-memory wavefronts per point = "
                   f"{float(d['l1tex__data_pipe_lsu_wavefronts_mem_shared.sum']) / pts:.2f}")
    out.append(f"thread-instructions per point = {32 * float(d['inst_executed']) / pts:.1f}")
    return "\n".join(out)


if __name__ == "__main__":
    res = []
    for arg in sys.argv[1:]:
        name, pts, alg = arg.split(":")
        res.append(block(name, int(float(pts)), float(alg)))
    print("\n\n".join(res))
