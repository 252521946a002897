"""Run bench.py over every BASELINE workload (device-resident value + kernel
time, no e2e / CPU legs) and write one JSON list: tools/sweep_json.py OUT."""
import json
import subprocess
import sys

WORKLOADS = ["cfg1", "cfg2", "cfg3", "cfg3-afps", "cfg3-fps", "cfg4",
             "cfg5-fps-2048", "cfg5-fps-4096", "cfg5-fps-8192", "cfg5-fps-16384", "cfg5-fps-32768",
             "cfg5-afps4-8192", "cfg5-afps16-8192", "cfg5-afps64-8192", "cfg5-afps256-8192",
             "cfg5-afps16-32768", "cfg5-afps256-32768", "cfg5-npdu-2048", "cfg5-npdu-8192",
             "cfg5-npdu-32768", "cfg5-1m"]


def main(out):
    rows = []
    for w in WORKLOADS:
        steps = "3" if w in ("cfg5-fps-16384", "cfg5-fps-32768") else "10"
        p = subprocess.run([sys.executable, "bench.py", "--workload", w, "--steps", steps,
                            "--warmup", "3", "--no-cpu-baseline", "--no-e2e"],
                           capture_output=True, text=True, timeout=900)
        line = [x for x in p.stdout.splitlines() if x.startswith("{")]
        if not line:
            rows.append({"workload": w, "error": p.stderr[-500:]})
            continue
        d = json.loads(line[-1])
        rows.append({"workload": w, "ms_per_step": d["ms_per_step"], "sampled_pts_per_s": d["value"],
                     "clouds_per_s": d["clouds_per_s"], "kernel": d["roofline"]["kernel"],
                     "kernel_ms": d["roofline"]["kernel_ms"], "fp64_frac": d["roofline"]["frac"],
                     "dist_evals_per_step": d["dist_evals_per_step"], "clocks": d["clocks"]})
        print(json.dumps(rows[-1]), flush=True)
    with open(out, "w") as f:
        json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1])
