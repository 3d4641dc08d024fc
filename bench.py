#!/usr/bin/env python
"""Benchmark of one Lloyd iteration (arXiv 2405.12052) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NS|C1..C5]
                    [--scaling strong|weak] [--impl ours|reference]

A "step" is one pass of the whole hot path over the workload: assign + fused
per-cluster reduction, deterministic merge, (NCCL allreduce when N > 1), and
the update (means, E, inertia, stop flag) -- SURVEY.md §8(a) rows a1-a9.
Inputs are resident in HBM before the timed region; W warm-up steps, then
exactly K steps between CUDA events on the context's stream, bracketed by a
barrier and a device synchronize, max over ranks.  The dataset (1.2 GB per
GPU at the default workload) is larger than the 126 MB L2, so no flush is
needed between steps.

For N > 1 launch with torchrun (one process per GPU); the library's own NCCL
communicator is created from a unique id broadcast over torch.distributed.

Prints ONE JSON line (rank 0).  See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import platform
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0      # /opt/skills/guides/B200_PROFILING.md fallback
SMS = 148
FP32_LANES_PER_SM = 128


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--workload", default="NS")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-iters", type=int, default=20)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--repeats", type=int, default=3,
                    help="timed repeats of exactly --steps steps each; the median is reported")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU time of the oracle baseline sample")
    ap.add_argument("--ref-seconds", type=float, default=60.0,
                    help="--impl reference: target CPU time of the whole run")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sort", action="store_true",
                    help="keep the caller's point order (full-scan assign kernel)")
    ap.add_argument("--no-fullscan-roofline", action="store_true")
    ap.add_argument("--gen", choices=["host", "device"], default="host",
                    help="where the synthetic shard is generated: datagen on the host, or "
                         "kmeans_generate in HBM (SURVEY.md NEXT-2; the e2e leg still copies "
                         "it to pinned host memory first, outside its timing)")
    ap.add_argument("--exchange", choices=["p2p", "nccl"], default="p2p",
                    help="P > 1: the per-iteration allreduce as one kernel over peer memory "
                         "(kmeans_p2p_open, default) or ncclAllReduce in the graph")
    return ap.parse_args()


def peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, 1965.0, "fallback"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor()


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML sampling thread)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.samples, self.reasons = [], 0
        self.period = period_s
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - depends on the box
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            time.sleep(self.period)

    def sample(self):
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            pass

    def __enter__(self):
        if self.ok:
            self.sample()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()
            self.sample()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU oracle baseline (rank 0, N = 1 only) and the reference arm
# ---------------------------------------------------------------------------
def oracle_points(w) -> int:
    """Prefix of the workload the oracle is timed on (both oracle legs use the
    same sample, so cpu_baseline and the reference arm agree): 8e6 points
    (96 MB, past the host caches) at K <= 16, 2e5 at K = 1024 (the oracle is
    exactly linear in N K)."""
    return min(w.N, 8_000_000 if w.K <= 16 else 200_000)


class PinnedCore:
    """Pins the calling thread to one host core (the oracle is single-threaded;
    `taskset -c <core>` equivalent) and restores the old mask afterwards."""

    def __enter__(self):
        self.old = os.sched_getaffinity(0)
        self.core = max(self.old)   # the highest allowed core (away from core 0's IRQs)
        os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *a):
        os.sched_setaffinity(0, self.old)


def oracle_run(w, iters: int, warmup: int = 1):
    """Times `iters` whole Lloyd iterations (oracle.step, the oracle as it
    stands, single thread pinned to one core) on oracle_points(w) points,
    after `warmup` untimed ones.  Returns per-iteration seconds."""
    import oracle
    from paper_2405_12052_b200 import datagen
    n = oracle_points(w)
    X = datagen.generate(w, 0, n, N=w.N)
    mu = X[datagen.init_indices(w, N=n, K=w.K)].astype(np.float64)
    times = []
    with PinnedCore() as pin:
        for _ in range(warmup):
            mu = oracle.step(X, mu)["mu_next"]
        for _ in range(iters):
            t0 = time.perf_counter()
            mu = oracle.step(X, mu)["mu_next"]
            times.append(time.perf_counter() - t0)
    return dict(n=n, times=times, core=pin.core)


def oracle_sample(w, target_s: float):
    """cpu_baseline: ~target_s seconds of oracle iterations (median per
    iteration, reported as points·iter/s)."""
    import oracle
    from paper_2405_12052_b200 import datagen
    n = oracle_points(w)
    X = datagen.generate(w, 0, min(n, 50_000), N=w.N)
    t0 = time.perf_counter()
    oracle.step(X, X[:w.K].astype(np.float64) + 0.5)
    per_iter = (time.perf_counter() - t0) * n / X.shape[0]
    iters = max(3, int(target_s / max(per_iter, 1e-9)))
    r = oracle_run(w, iters)
    med = statistics.median(r["times"])
    return dict(value=r["n"] / med, n=r["n"], iters=iters, seconds=sum(r["times"]),
                core=r["core"])


def run_reference(args, w):
    """The reference arm: the oracle as it stands (there is no reference
    implementation -- /root/reference is a paper), one whole Lloyd iteration
    per step on the oracle_points(w)-point prefix of the same workload,
    single thread pinned to one core; ms_per_step is the sample's own."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0  # under torchrun only rank 0 runs the oracle
    r = oracle_run(w, args.steps, warmup=args.warmup)
    n = r["n"]
    dt = sum(r["times"])
    value = n * args.steps / dt
    sample = (f"{n} of {w.N} points (prefix of the seeded {w.name} workload), "
              f"{args.steps} whole Lloyd iterations (oracle.step) after {args.warmup} warm-up, "
              f"single thread pinned to core {r['core']}; ms_per_step is this sample's")
    line = {
        "impl": "reference", "metric": "Lloyd points·iter/s", "value": value,
        "unit": "points·iter/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": dict(workload_config(w, args.gpus, args.scaling), gen=args.gen,
                       **({"exchange": args.exchange} if args.gpus > 1 else {})),
        "sample_points": n,
        "cpu_baseline": {"value": value, "unit": "points·iter/s", "cores": 1,
                         "kind": "oracle", "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "points·iter/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(w, P, scaling):
    per_gpu = w.N // P if scaling == "strong" else w.N
    return {"workload": w.name, "N": w.N if scaling == "strong" else w.N * P, "d": w.d,
            "K": w.K, "per_gpu_N": per_gpu, "blobs": w.M, "tol": 0.0,
            "parallelism": f"dp{P}",
            "l2": f"inputs larger than L2 ({per_gpu * w.d * 4 / 1e6:.0f} MB per GPU vs 126 MB)"
            if per_gpu * w.d * 4 > 126e6 else "inputs fit in L2 (no flush)"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def main():
    args = parse()
    from paper_2405_12052_b200 import datagen
    w = datagen.WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args, w)

    import torch
    import torch.distributed as dist
    from paper_2405_12052_b200 import kmeans as km

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    P = world
    assert P == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    distributed = P > 1
    comm = None
    if distributed:
        from paper_2405_12052_b200 import dist as kdist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = kdist.init_comm(rank, P, local)

    def barrier():
        if distributed:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if not distributed:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # shard (contiguous ceiling partition, PAPER.md:97 / SPEC.md:236)
    global_N = w.N if args.scaling == "strong" else w.N * P
    from paper_2405_12052_b200 import dist as kdist_
    a, b = kdist_.shard(global_N, P, rank)   # ValueError on every rank if a shard is empty
    gen_w = w if args.scaling == "strong" else dataclasses.replace(w, N=global_N)
    Xh = torch.empty((b - a, w.d), dtype=torch.float32, pin_memory=True)
    Xd = None
    if args.gen == "device":
        Xd = torch.empty((b - a, w.d), dtype=torch.float32, device="cuda")
        km.generate(datagen.mixture_spec(gen_w, global_N), a, b - a, Xd, device=local)
        Xh.copy_(Xd)
    else:
        datagen.generate(gen_w, a, b - a, N=global_N, out=Xh.numpy())
    init = datagen.init_indices(gen_w, N=global_N, K=w.K)

    exchange = {"mode": args.exchange if distributed else "none"}

    def make_ctx(points, sort, expected_iters=0):
        c = km.Context(points, w.K, device=local, comm=comm, global_offset=a, global_N=global_N,
                       sort=sort, expected_iters=expected_iters)
        if distributed and args.exchange == "p2p":
            # collective: all-gathers the IPC handles; all ranks fall back to
            # the NCCL allreduce if any rank cannot map its peers
            if not kdist.enable_p2p(c):
                exchange["mode"] = "nccl (p2p mapping unavailable)"
        return c

    # (the timed context measures steady-state throughput: the library's
    # default path choice, no iteration-count hint; the e2e leg below passes
    # its own iteration count)
    ctx = make_ctx(Xh if Xd is None else Xd, False if args.no_sort else None)
    del Xd   # the context holds its own (sorted) copy
    info = ctx.info()
    stream = torch.cuda.ExternalStream(ctx.stream)
    ctx.start(init_idx=init, tol=0.0, max_iter=1 << 30)

    # warm-up (also instantiates the CUDA graph)
    ctx.iterate(args.warmup)
    ctx.poll()
    barrier()
    # the dominant kernel alone, once right before the timed region (GPU warm);
    # again right after it (see below) -- the roofline uses the mean of the two
    one_kernel = bool(info["fused"] or info["persistent"])   # the iteration is one kernel
    pre_assign = (None if one_kernel else
                  ctx.profile_stage(max(20, min(args.steps, 200)), 1, timed=True) / 1e3)

    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    rep_ms = []
    launches_per_rep = []
    with ClockSampler(local) as clocks:
        for _ in range(args.repeats):   # each repeat: exactly K steps between barriers
            launches0 = ctx.info()["kernel_launches"]
            barrier()
            e0.record(stream)
            ctx.iterate(args.steps)
            e1.record(stream)
            e1.synchronize()
            barrier()
            launches_per_rep.append(ctx.info()["kernel_launches"] - launches0)
            rep_ms.append(max_over_ranks(e0.elapsed_time(e1)))
    ms = statistics.median(rep_ms)
    launches = launches_per_rep[rep_ms.index(ms)] if ms in rep_ms else launches_per_rep[0]
    st = ctx.poll()
    assert st["iters"] == args.warmup + args.repeats * args.steps, st

    value = global_N * args.steps / (ms / 1e3)   # whole-job points·iter/s
    ms_per_step = ms / args.steps

    # ---- dominant kernel alone (roofline): assign + fused reduction ------------
    def time_assign(c, stage=1):
        # stage 1: the assign kernels alone (kmeans_profile_stage): `reps`
        # launches captured in one CUDA graph, CUDA events on the library's
        # stream around the graph launch -> device ms per launch
        reps = max(20, min(args.steps, 200))
        return c.profile_stage(reps, stage, timed=True) / 1e3   # s per launch

    n_local = b - a
    hbm_gbs, sm_max_mhz, peak_src = peaks()
    clk = clocks.summary()
    bytes_per_launch = 4.0 * w.d * n_local                      # read every point once
    lane_ops_per_launch = 2.0 * w.d * w.K * n_local             # form D: d FADD, 1 FMUL, d-1 FFMA
    fp32_peak = SMS * FP32_LANES_PER_SM * sm_max_mhz * 1e6 / 1e12   # T lane-ops/s
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(f"{w.name}:P{P}:{args.scaling}:{'sorted' if info['sorted'] else 'unsorted'}")
    except Exception:
        pass

    def roofline_of(t_kernel, kernel, sorted_path):
        ach_gbs = bytes_per_launch / t_kernel / 1e9
        ach_tops = lane_ops_per_launch / t_kernel / 1e12
        common = {"kernel": kernel, "kernel_ms": t_kernel * 1e3,
                  "kernel_share_of_step": t_kernel * 1e3 / ms_per_step}
        t_hbm = bytes_per_launch / (hbm_gbs * 1e9)
        t_alu = lane_ops_per_launch / (fp32_peak * 1e12)
        if sorted_path or t_hbm >= t_alu:
            # the pruned kernel does not perform the full 2dK FP32 work: its
            # binding roofline is the HBM stream of the points
            return dict(bound="hbm", achieved=ach_gbs, peak=hbm_gbs, unit="GB/s",
                        frac=ach_gbs / hbm_gbs, traffic=traffic,
                        frac_of_8tbs_spec=ach_gbs / 8000.0,
                        peak_source=f"MEASURED_PEAKS.json hbm_gbs ({peak_src})", **common)
        return dict(bound="alu", achieved=ach_tops, peak=fp32_peak, unit="TFLOP/s",
                    op="FP32 lane-op (FADD, FMUL, FFMA = 1 each)", frac=ach_tops / fp32_peak,
                    traffic=traffic, peak_source=f"148 SMs x 128 FP32 lanes x {sm_max_mhz:.0f} MHz",
                    hbm_frac=ach_gbs / hbm_gbs, **common)

    if one_kernel:
        # the whole iteration is ONE kernel, many iterations per cooperative
        # launch (k_fused_iterate: small full-scan shards; k_persist_iterate:
        # the sorted small-K path) -- its time per iteration is the step
        t_assign = ms_per_step / 1e3
        kname = "k_fused_iterate" if info["fused"] else "k_persist_iterate"
        stage_ms = {"iteration": ms_per_step}
        if info["persistent"]:
            # for reference: the multi-kernel path's assign kernel and row merge alone
            stage_ms["k_assign_pruned_alone"] = time_assign(ctx) * 1e3
            stage_ms["row_merge_alone"] = time_assign(ctx, 2) * 1e3
    else:
        post_assign = time_assign(ctx)
        # kernel time "around" the timed region: the mean of the measurements
        # right before and right after it (clocks drift under sustained load)
        t_assign = 0.5 * (pre_assign + post_assign)
        if info["sorted"]:
            kname = ("k_assign_pruned" if info["path"] == 0
                     else "k_prune+k_assign_pruned+k_assign_heavy_tiles")
        else:
            kname = "k_assign_chunk" if info["path"] == 0 else "k_assign_large"
        # per-stage device time (each stage alone, back-to-back launches)
        stage_ms = {"assign": t_assign * 1e3, "assign_before": pre_assign * 1e3,
                    "assign_after": post_assign * 1e3, "row_merge": time_assign(ctx, 2) * 1e3}
        stage_ms["merge_update_and_gaps"] = ms_per_step - stage_ms["assign"] - stage_ms["row_merge"]
        stage_ms["k_merge_alone"] = time_assign(ctx, 3) * 1e3   # the P>1 path's group merge
    roofline = roofline_of(t_assign, kname, bool(info["sorted"]))
    roofline_hbm = {"achieved": bytes_per_launch / t_assign / 1e9, "peak": hbm_gbs, "unit": "GB/s",
                    "frac": bytes_per_launch / t_assign / 1e9 / hbm_gbs,
                    "step_frac": (bytes_per_launch / (ms_per_step / 1e3) / 1e9) / hbm_gbs,
                    "peak_source": peak_src}
    cand = ctx.candidate_stats() if info["sorted"] else None
    fullscan = None
    if info["sorted"] and not args.no_fullscan_roofline:
        # the same shard through the full-scan kernel (caller's order, no pruning)
        cf = make_ctx(Xh, False)
        cf.start(init_idx=init, tol=0.0, max_iter=1 << 30)
        tf = time_assign(cf)
        fullscan = roofline_of(tf, "k_assign_chunk" if w.K <= 16 else "k_assign_large", False)
        cf.close()

    # ---- end to end through the public API with host buffers ------------------------
    e2e = None
    if not args.no_e2e:
        labels_h = torch.empty(n_local, dtype=torch.int32, pin_memory=True)
        ctx.close()

        def e2e_run(sort):
            def e2e_step():
                barrier()
                t0 = time.perf_counter()
                c2 = make_ctx(Xh, sort, expected_iters=args.e2e_iters)
                t1 = time.perf_counter()
                r = c2.fit(init, 0.0, args.e2e_iters, out_labels=labels_h, traces=False)
                t2 = time.perf_counter()
                srt = c2.info()["sorted"]
                c2.close()
                t3 = time.perf_counter()
                barrier()
                assert r["iters"] == args.e2e_iters
                return max_over_ranks(t3 - t0), (t1 - t0, t2 - t1, t3 - t2), srt

            e2e_step()   # warm-up step (first-use costs: allocations, module loading)
            steps = [e2e_step() for _ in range(args.e2e_steps)]
            dts = sorted(x[0] for x in steps)
            dt = statistics.median(dts)
            parts = [statistics.median(x[1][i] for x in steps) for i in range(3)]
            return {"value": global_N * args.e2e_iters / dt, "unit": "points·iter/s",
                    "h2d_bytes_per_step": int(Xh.numel() * 4 + 8 * w.K),
                    "d2h_bytes_per_step": int(n_local * 4 + 8 * w.K * w.d + 16),
                    "step": f"one kmeans_create (opts.expected_iters = {args.e2e_iters}) + "
                            f"kmeans_fit_ctx ({args.e2e_iters} iterations, labels out) + "
                            "kmeans_destroy call from pinned host memory",
                    "steps_timed": args.e2e_steps, "warmup_steps": 1,
                    "seconds_per_step": dt, "sorted": steps[0][2],
                    "breakdown_s": {"create": parts[0], "fit": parts[1], "destroy": parts[2]}}

        # the library's own path choice (the call a user makes) ...
        e2e = e2e_run(False if args.no_sort else None)
        # ... and the other path beside it, for reference
        alt = e2e_run(bool(not e2e["sorted"]))
        e2e["other_path"] = {"sorted": alt["sorted"], "value": alt["value"],
                             "seconds_per_step": alt["seconds_per_step"],
                             "breakdown_s": alt["breakdown_s"]}
    else:
        ctx.close()

    cpu = None
    if rank == 0 and P == 1 and not args.no_cpu_baseline:
        s = oracle_sample(w, args.cpu_seconds)
        cpu = {"value": s["value"], "unit": "points·iter/s", "cores": 1, "kind": "oracle",
               "sample": f"{s['iters']} Lloyd iterations (oracle.step) on the first {s['n']} "
                         f"points of {w.name}, single-threaded C oracle pinned to core "
                         f"{s['core']}, {s['seconds']:.1f} s, median iteration",
               "cpu": cpu_model(), "host_cores": os.cpu_count()}

    if distributed:
        km.comm_destroy(comm)
    if rank == 0:
        line = {
            "metric": "Lloyd points·iter/s", "value": value, "unit": "points·iter/s",
            "n_gpus": P, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "repeats_ms_per_step": [m / args.steps for m in rep_ms], "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(workload_config(w, P, args.scaling), gen=args.gen,
                           **({"exchange": exchange["mode"]} if P > 1 else {})),
            "roofline": roofline, "roofline_hbm": roofline_hbm, "stage_ms": stage_ms,
            "roofline_fullscan": fullscan, "candidates": cand,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "kernels_per_step": info["kernels_per_iter"],
            "clocks": clk,
            "launch": ({"grid": info["persist_grid"], "kernel": "k_persist_iterate",
                        "sorted": 1, "persistent": 1} if info["persistent"] else
                       {"grid": info["grid"], "block": info["block"],
                        "smem_bytes": info["smem_bytes"], "path": info["path"],
                        "sorted": info["sorted"]}),
        }
        print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
