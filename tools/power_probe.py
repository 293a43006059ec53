"""Runs tools/power_probe for a few operating points and samples board power
and SM clock (nvidia-smi) during each: the (fp32 rate, HBM rate, power, clock)
points behind DESIGN's power model. Output: JSON lines."""
import json
import statistics
import subprocess
import sys
import threading
import time

POINTS = [("idle", 100), ("fp", 100), ("fp", 50), ("lds", 100), ("mov", 100), ("l2", 100), ("copy", 100),
          ("both", 100), ("both", 50)]


def sample(stop, out):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=power.draw,clocks.sm,clocks_throttle_reasons.sw_power_cap",
                            "--format=csv,noheader,nounits"], capture_output=True, text=True)
        try:
            p, c, cap = [x.strip() for x in r.stdout.strip().split(",")]
            out.append((float(p), float(c), cap))
        except Exception:
            pass
        time.sleep(0.2)


def main():
    secs = sys.argv[1] if len(sys.argv) > 1 else "6"
    only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
    for mode, duty in POINTS:
        if only and mode not in only:
            continue
        stop, samples = threading.Event(), []
        th = threading.Thread(target=sample, args=(stop, samples))
        th.start()
        if mode == "idle":
            time.sleep(float(secs))
            r = subprocess.CompletedProcess([], 0, '{"probe": "power", "mode": "idle"}\n', "")
        else:
            r = subprocess.run(["tools/power_probe", mode, secs, str(duty)], capture_output=True, text=True)
        stop.set()
        th.join()
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        d = json.loads(line[-1]) if line else {"error": r.stderr[-300:]}
        tail = samples[len(samples) // 3:]  # after the limiter has settled
        if tail:
            d["power_w_median"] = statistics.median(s[0] for s in tail)
            d["sm_mhz_median"] = statistics.median(s[1] for s in tail)
            d["sw_power_cap_active"] = sum(1 for s in tail if "Active" in s[2] and "Not" not in s[2]) / len(tail)
        print(json.dumps(d), flush=True)
        time.sleep(2)


if __name__ == "__main__":
    main()
