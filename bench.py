"""Benchmark: FPS / AFPS / NPDU-AFPS sampling throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference      # the reference CPU path, same config

Metric (BASELINE.json): sampled points/s (and clouds/s), whole job. A step is
one pass of the hot path over one batch resident in HBM: the per-cloud stable
axis sort (when the config sorts) plus the sampler, both hand-written sm_100a
kernels. Weak scaling: every rank samples its own batch of the configured
size (clouds are independent, no collective on the data path). Timing: CUDA
events on the launching stream around each step, an L2 flush (a 512 MiB
write, > 126 MB L2) between steps outside the events, barrier + synchronize on
both sides of the K timed steps, max over ranks.

Also reported: `e2e` (the same metric through the public API with host
buffers: pinned H2D of the batch, sort + sample, D2H of indices + stats, every
step), `roofline` (the sampler kernel's FP64 work against the measured FP64
peak), `cpu_baseline` (the unmodified reference, oracle/_ref, on this host's
cores, bounded sample), `clocks` (nvidia-smi during the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Per-GPU workloads (BASELINE.json configs; BASELINE's w -> k = 2w + 1).
WORKLOADS = {
    "cfg1": dict(gen="cube", B=1, N=2048, method="fps", C=512, M=1, K=None, sort="x"),
    "cfg2": dict(gen="prim4", B=16, N=2048, method="afps", C=512, M=8, K=None, sort="x"),
    "cfg3": dict(gen="prim6", B=64, N=8192, method="npdu_afps", C=2048, M=16, K=65, sort="x"),
    "cfg3-afps": dict(gen="prim6", B=64, N=8192, method="afps", C=2048, M=16, K=None, sort="x"),
    "cfg3-fps": dict(gen="prim6", B=64, N=8192, method="fps", C=2048, M=1, K=None, sort="x"),
    "cfg4": dict(gen="lidar", B=128, N=32768, method="npdu_afps", C=8192, M=32, K=129, sort=None),
}
for _n in (2048, 4096, 8192, 16384, 32768):
    WORKLOADS[f"cfg5-fps-{_n}"] = dict(gen="cube", B=256, N=_n, method="fps", C=_n // 4, M=1,
                                       K=None, sort="x")
    for _m in (4, 16, 64, 256):
        WORKLOADS[f"cfg5-afps{_m}-{_n}"] = dict(gen="cube", B=256, N=_n, method="afps",
                                                C=_n // 4, M=_m, K=None, sort="x")
    WORKLOADS[f"cfg5-npdu-{_n}"] = dict(gen="cube", B=256, N=_n, method="npdu_afps", C=_n // 4,
                                        M=16, K=65, sort="x")

# one 1M-point cloud: under torchrun its sectors are split across the ranks
# (strong scaling, BASELINE cfg5), each rank sorting the cloud itself
WORKLOADS["cfg5-1m"] = dict(gen="cube", B=1, N=1 << 20, method="afps", C=(1 << 20) // 4, M=1024,
                            K=None, sort="x", strong=True)

# latency probes: one NPDU sector per warp, 1 warp / 148 warps / 4096 warps
for _b in (1, 148, 4096):
    WORKLOADS[f"lat-npdu-{_b}"] = dict(gen="cube", B=_b, N=1024, method="npdu_fps", C=256, M=1,
                                       K=129, sort=None)

DEFAULT_WORKLOAD = "cfg4"
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peak.json")


def make_input(w, seed_base=0):
    from paper_2208_08795_b200 import synth

    g = w["gen"]
    if g == "cube":
        return synth.uniform_cube(w["B"], w["N"], seed_base)
    if g.startswith("prim"):
        return synth.primitives(w["B"], w["N"], int(g[4:]), seed=seed_base + 1)
    if g == "lidar":
        return synth.lidar_sweep(w["B"], seed=seed_base + 4)
    raise ValueError(g)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 3:
                try:
                    self.rows.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        loaded = [r for r in self.rows if not (r[2] & 0x1)] or self.rows
        mask = 0
        for r in loaded:
            mask |= r[2]
        return {"sm_mhz": float(np.median([r[0] for r in loaded])),
                "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": [v for k, v in self.REASONS.items() if mask & k and k != 0x1],
                "samples": len(loaded)}


def ncu_traffic(workload):
    """DRAM bytes per launch of the sampler kernel (and its issue rate) from
    the committed ncu --set full summary for this workload
    (profiles/ncu_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)[workload]
        return float(d["dram_bytes"]), d["source"], d.get("ipc_per_sm")
    except (OSError, KeyError, ValueError):
        return None, "no ncu capture for this workload", None


def fp64_peak():
    try:
        with open(FP64_PEAK_FILE) as f:
            d = json.load(f)
        return float(d["fp64_tflops"]), d.get("source", FP64_PEAK_FILE)
    except (OSError, KeyError, ValueError):
        return None, "missing"


def cpu_reference(w, xyz_sorted, budget_s=20.0, steps=1, quiet=False):
    """The unmodified reference (oracle/_ref) on the host: one cloud per
    worker thread, sampler at threads=1 (proj/src/bench.cpp:90-92,104-120),
    timed around the sampler calls only, best of `steps` runs. Bounded: a
    prefix of the batch sized to ~budget_s of single-core work."""
    from oracle import Reference

    ref = Reference()
    workers = os.cpu_count() or 1
    probe = xyz_sorted[:1]
    _, _, t1 = ref.sample_batch_f32(w["method"], probe, w["C"], w["M"], w["K"] or 0, workers=1)
    per_cloud = max(t1, 1e-6)
    nb = int(max(1, min(w["B"], budget_s / per_cloud)))
    nb = max(min(nb, w["B"]), min(w["B"], workers))
    sample = xyz_sorted[:nb]
    best = None
    for _ in range(max(1, steps)):
        _, _, secs = ref.sample_batch_f32(w["method"], sample, w["C"], w["M"], w["K"] or 0,
                                          workers=workers)
        best = secs if best is None else min(best, secs)
    pts_s = nb * w["C"] / best
    return {"value": pts_s, "unit": "sampled points/s", "cores": min(workers, nb),
            "kind": "reference", "clouds_per_s": nb / best,
            "sample": f"{nb} of {w['B']} clouds of the same batch (pre-sorted on the host), "
                      f"{min(workers, nb)} worker threads, best of {max(1, steps)}, "
                      f"single-core probe {per_cloud * 1e3:.2f} ms/cloud",
            "cpu_model": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def launches_per_step(w):
    """Our kernels per step (csrc/sort_kernels.cu, csrc/sample_dispatch.cu):
    one sampler launch; the axis sort is one launch up to 256K fp32 points,
    otherwise the device-wide radix (histogram, scan, scatter per 8-bit
    pass)."""
    sort = 0
    if w["sort"]:
        sort = 1 if w["N"] <= 16 * 16384 else 3 * 4
    return 1 + sort


def host_sorted(w, xyz):
    if w["sort"] is None:
        return xyz
    from paper_2208_08795_b200 import synth

    return synth.stable_sort_np(xyz, "xyz".index(w["sort"]))[0]


def arm_config(workload, w, world, strong):
    """The `config` object both arms print (identical for the same workload)."""
    return {"workload": workload, "clouds_per_gpu": w["B"], "points_per_cloud": w["N"],
            "samples_per_cloud": w["C"], "method": w["method"], "m": w["M"], "k": w["K"],
            "sort": w["sort"], "generator": w["gen"], "coords": "fp32 in, fp64 math",
            "l2": "flushed between steps (512 MiB write)",
            "parallelism": (f"sector-split x{world}" if strong else f"dp{world}")}


def run_reference_arm(args, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    xyz = make_input(w)
    res = cpu_reference(w, host_sorted(w, xyz), budget_s=8.0, steps=args.steps)
    line = {"metric": "sampled points/s", "value": res["value"], "unit": "sampled points/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": arm_config(args.workload, w, args.gpus,
                                 bool(w.get("strong")) and args.gpus > 1),
            "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "clouds_per_s": res["clouds_per_s"], "cpu_model": res["cpu_model"],
            "e2e": {"value": res["value"], "unit": "sampled points/s",
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference_arm(args, w)

    import torch
    import torch.distributed as dist

    import paper_2208_08795_b200 as pcs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    args.warmup = max(args.warmup, 3)

    # weak scaling: each rank gets its own clouds (seeded by rank); strong
    # (one cloud, world > 1): every rank holds the same cloud, sorts it, and
    # samples its contiguous run of sectors with global index / sector bases
    strong = bool(w.get("strong")) and world > 1
    xyz_host = make_input(w, seed_base=0 if strong else 1000 * rank)
    xyz = torch.from_numpy(xyz_host).to(dev)
    B, N, C = w["B"], w["N"], w["C"]
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    from paper_2208_08795_b200 import shard

    sh = shard.sector_shard(N, C, w["M"], world, rank) if strong else None

    def sample_sorted(xs):
        if sh is None:
            return pcs.sample(xs, C, method=w["method"], m=w["M"], k=w["K"])
        return pcs.sample(xs[:, sh.point_lo:sh.point_hi], sh.c, method=w["method"], m=sh.m,
                          k=w["K"], index_base=sh.point_lo, sector_base=sh.sector_lo)

    def step(x):
        if sh is None:
            return pcs.sample(x, C, method=w["method"], m=w["M"], k=w["K"], sort=w["sort"])
        xs = pcs.sort_axis(x, w["sort"])[0] if w["sort"] else x
        return sample_sorted(xs)

    for _ in range(args.warmup):
        out = step(xyz)
    torch.cuda.synchronize()
    stats = out[1].cpu().numpy()
    evals_per_step = int(stats[:, 0].sum())

    # ---- device-resident throughput (value)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            flush.fill_(float(i))
            starts[i].record()
            step(xyz)
            ends[i].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_per_step = ms / args.steps
    total_samples = B * C if strong else world * B * C
    pts_per_s = total_samples / (ms_per_step * 1e-3)

    # ---- sampler kernel alone (roofline): sort once, time only the sampler
    xs = pcs.sort_axis(xyz, w["sort"])[0] if w["sort"] else xyz
    ks, ke = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kern_ms = 0.0
    for i in range(args.steps):
        flush.fill_(float(i))
        ks.record()
        sample_sorted(xs)
        ke.record()
        torch.cuda.synchronize()
        kern_ms += ks.elapsed_time(ke)
    kern_ms /= args.steps
    peak, peak_src = fp64_peak()
    flops = 8.0 * evals_per_step
    achieved = flops / (kern_ms * 1e-3) / 1e12
    traffic, traffic_src, ipc = ncu_traffic(args.workload)
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if peak else None, "traffic": traffic,
                "traffic_source": traffic_src,
                # what actually limits the serial update->argmax->pivot chain:
                # issued instructions per SM-cycle (ncu) against the 4 schedulers
                "issue": ({"ipc_per_sm": ipc, "peak_ipc": 4.0, "frac": ipc / 4.0}
                          if ipc else None),
                "algorithmic_hbm_bytes": B * N * 12 + B * C * 4,
                "kernel": pcs.kernel_family(w["method"], N, w["M"], w["K"], batch=B),
                "kernel_ms": kern_ms, "algorithmic_flops": flops, "peak_source": peak_src,
                "note": "FP64 flops = 8 x dist_evals (3 sub, 3 mul, 2 add; no FMA); the "
                        "argmax work is not counted"}

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        pinned = torch.from_numpy(xyz_host).pin_memory()

        def e2e_step():
            # the C-ABI host-buffer entry (pcs_sample_host_batch, through
            # pcs.sample_host_batch): pinned batch in, host results out,
            # chunked H2D / sort + sample / D2H inside the native call
            if sh is None:
                return pcs.sample_host_batch(pinned, C, method=w["method"], m=w["M"], k=w["K"],
                                             sort=w["sort"])
            res = step(pinned.to(dev, non_blocking=True))
            return tuple(t.cpu() for t in res)

        # warm-up: at least W steps and 0.5 s -- the host link ramps up over
        # the first ~15 transfers after idling (1.6-3 ms -> 1.2 ms per step
        # measured, tools/e2e_dbg.py)
        t_warm = time.perf_counter()
        for i in range(max(args.warmup, 1000)):
            e2e_step()
            if i + 1 >= args.warmup and time.perf_counter() - t_warm > 0.5:
                break
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_ms = 0.0
        for i in range(args.steps):
            flush.fill_(float(i))
            es.record()
            e2e_step()
            ee.record()
            torch.cuda.synchronize()
            e_ms += es.elapsed_time(ee)
        t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item()) / args.steps
        r = e2e_step()
        # the PCIe floor on this box: one plain H2D of the same pinned batch
        dst = torch.empty(pinned.shape, dtype=pinned.dtype, device=dev)
        h2d = []
        for _ in range(5):
            es.record()
            dst.copy_(pinned, non_blocking=True)
            ee.record()
            torch.cuda.synchronize()
            h2d.append(es.elapsed_time(ee))
        del dst
        e2e = {"value": total_samples / (e_ms * 1e-3), "unit": "sampled points/s",
               "ms_per_step": e_ms, "h2d_floor_ms": min(h2d),
               "h2d_gbps": pinned.numel() * pinned.element_size() / min(h2d) / 1e6,
               "h2d_bytes_per_step": int(pinned.numel() * pinned.element_size()),
               "d2h_bytes_per_step": int(sum(t.nbytes if hasattr(t, "nbytes") else
                                             t.numel() * t.element_size() for t in r)),
               "path": ("C-ABI pcs_sample_host_batch (pinned host tensor in, host arrays out): "
                        "chunked H2D overlapped with sort+sample, D2H of indices, stats (and "
                        "perm when sorting)") if sh is None else
                       "pinned H2D, sort, sample of this rank's sectors, D2H"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_reference(w, host_sorted(w, xyz_host))
            cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model")}
        except Exception as exc:  # the checker is optional on the box
            cpu = {"value": None, "unit": "sampled points/s", "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": "sampled points/s", "value": pts_per_s, "unit": "sampled points/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "clouds_per_s": (B if strong else world * B) / (ms_per_step * 1e-3),
            "config": arm_config(args.workload, w, world, strong),
            "gpu_launches": args.steps * launches_per_step(w),
            "dist_evals_per_step": evals_per_step,
            "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
