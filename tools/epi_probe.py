import os, sys, statistics, json
sys.path.insert(0, os.getcwd())
import bench
import paper_1609_03361_b200 as sf
model, v, vmin = bench.make_model("c2")
s = sf.acoustic_build(model, True, v_field=v, v_min=vmin)
s.op.upload(); s.op.run(0, model.nt); s.op.synchronize()
full, sten = [], []
for _ in range(10):
    t, _, _ = s.op.time(stencil=False); full.append(t / model.nt * 1e3)
    t, st, _ = s.op.time(stencil=True); sten.append(st / model.nt * 1e3)
print(json.dumps({"full_us_per_step": statistics.median(full), "stencil_only_us_per_launch": statistics.median(sten)}))
