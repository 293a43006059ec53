import csv, sys
def summ(name, pts, algb):
    rr = list(csv.reader(open(f"gpurun_out/prof/{name}.raw.csv")))
    d = dict(zip(rr[0], rr[2])); u = dict(zip(rr[0], rr[1]))
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "inst_executed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"]
    out = [f"## {name}"]
    for k in keys:
        if k in d: out.append(f"{k} = {d[k]} {u.get(k,'')}".rstrip())
    sc = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}
    tot = float(d["dram__bytes_read.sum"]) * sc[u["dram__bytes_read.sum"]] + float(d["dram__bytes_write.sum"]) * sc[u["dram__bytes_write.sum"]]
    out.append(f"DRAM bytes per launch = {tot/1e6:.1f} MB; algorithmic = {algb/1e6:.1f} MB ({tot/algb:.3f}x)")
    out.append(f"thread-instructions per point (all lanes) = {32*float(d['inst_executed'])/pts:.1f}")
    return "\n".join(out), tot
res = []
tr = {}
for name, pts, algb in [("vec_c2", 277**3, 20*277**3), ("vec_c3o8", 504**3, 20*504**3), ("vecq_c3o16", 496**3, 20*496**3), ("tb_c1", 2046**2*8, 8*2046**2*8)]:
    s, tot = summ(name, pts, algb); res.append(s); tr[name] = tot
print("\n\n".join(res))
import json
json.dump({"c2": tr["vec_c2"], "c3o8": tr["vec_c3o8"], "c3o16": tr["vecq_c3o16"], "c1_per_8_steps": tr["tb_c1"]}, open("profiles/traffic.json","w"), indent=1)
