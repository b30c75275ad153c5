"""Benchmark of the B200 tiled QR hot path (BASELINE.json metric and configs[1]).

A step = one tiled QR factorization of the configs[1] matrix (8000 x 2000 fp64,
i.i.d. N(0,1), p=40 x q=10 tiles of nb=200, ib=32) with EACH tree in turn —
FlatTree (Sameh-Kuck), Fibonacci, Greedy, PlasmaTree BS=1,5,10,20 — and each
kernel family (TT and TS, Algorithms 3 and 2).
value = 2n^2(m-n/3) flops x cases x ranks / device time (GFLOP/s).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Multi-GPU (torchrun): every rank factors its own matrix (replicas, weak
scaling) — the cross-GPU TT merge of configs[3] is a separate row.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

P, Q, NB, IB = 40, 10, 200, 32
M, N = P * NB, Q * NB
TREES = [("flat", 1), ("fibonacci", 1), ("greedy", 1), ("plasma", 1), ("plasma", 5), ("plasma", 10),
         ("plasma", 20)]
FAMILIES = ("TT", "TS")          # north_star: "executed with TT (triangle-on-triangle) and TS tile kernels"
CASES = [(t, b, f) for f in FAMILIES for (t, b) in TREES]
FLOPS = 2.0 * N * N * (M - N / 3.0)
METRIC = "tiled QR fp64 GFLOP/s (2n²(m−n/3)) and % of B200 FP64 tensor peak, 1/2/4/8 GPU"
WORKLOAD = ("configs[1]: fp64 tiled QR 8000x2000 (p=40 x q=10 tiles, nb=200, ib=32), i.i.d. N(0,1), "
            "each tree in turn (flat, fibonacci, greedy, plasma BS=1,5,10,20) with TT and with TS kernels")
SEED = 2024


def fp64_peak():
    """FP64 tensor peak = measured bf16 burst peak x the guide's nominal FP64/bf16 ratio (45/2250)."""
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return mp["bf16_tflops"] * 45.0 / 2250.0, "MEASURED_PEAKS.json bf16_tflops x 45/2250 (guide nominal FP64/bf16)"
    except Exception:
        return 1590.0 * 45.0 / 2250.0, "fallback 1.59 PFLOP/s bf16 x 45/2250 (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler running during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, idx):
        self.idx = idx
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], 0, set()
        for line in (getattr(self, "out", "") or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic():
    """Per-launch DRAM bytes of tqr_persistent from the committed ncu --set full summary (or None)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_full_summary.json")))
        return d.get("dram_bytes_per_launch")
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU oracle legs (cpu_baseline and --impl reference): the oracle as it stands
# ---------------------------------------------------------------------------
def oracle_sample(budget_s: float, seed: int = SEED):
    """Run the oracle's tiled QR of the configs[1] Greedy factorization task by task
    (oracle/numeric.py kernels in dag.expand order) until `budget_s` seconds have
    passed; return (GFLOP/s, flops done, tasks done, threads)."""
    import qrinputs
    from oracle import dag, numeric as nu, schemes
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        threads = 1
    A = qrinputs.gaussian(M, N, seed)
    lst = schemes.elim_list("greedy", P, Q)
    F = nu.Factor(np.array(A, order="F"), P, Q, NB, IB, dag.expand(lst, P, Q, "TT"))
    unit = NB ** 3 / 3.0
    done_flops, ntask = 0.0, 0
    t0 = time.perf_counter()
    for t in F.tasks:
        if t.kind == "GEQRT":
            taus, Tm = nu.geqrt(F.tile(t.i, t.k), IB)
            F.tau[(0, t.i, t.k)] = taus
        elif t.kind == "UNMQR":
            nu.unmqr(F.tile(t.i, t.k), F.tau[(0, t.i, t.k)], F.tile(t.i, t.j))
        elif t.kind == "TTQRT":
            taus, Tm = nu.ttqrt(F.tile(t.piv, t.k), F.tile(t.i, t.k), IB)
            F.tau[(1, t.i, t.k)] = taus
        else:
            nu.ttmqr(F.tile(t.i, t.k), F.tau[(1, t.i, t.k)], F.tile(t.piv, t.j), F.tile(t.i, t.j))
        done_flops += t.weight * unit
        ntask += 1
        if time.perf_counter() - t0 > budget_s:
            break
    el = time.perf_counter() - t0
    return done_flops / el / 1e9, done_flops, ntask, len(F.tasks), threads, el


def run_reference(args, rank, world):
    if rank != 0:
        return
    budget = float(os.environ.get("TQR_REF_BUDGET_S", "8"))
    vals = []
    for _ in range(args.warmup):
        oracle_sample(min(budget, 2.0))
    for _ in range(args.steps):
        g, fl, nt, tot, thr, el = oracle_sample(budget)
        vals.append(g)
    v = float(np.mean(vals))
    sample = (f"first {nt} of {tot} tasks (in list order) of the Greedy TT factorization of configs[1], "
              f"{budget:.0f} s budget per step, oracle/numeric.py kernels (numpy fp64)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": budget * 1000.0, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample": sample},
        "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": thr, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------
def run_gpu(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_1104_4475_b200 as tq

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.Stream(device=dev)
    rng = np.random.Generator(np.random.PCG64(SEED + rank))
    A_host = np.ascontiguousarray(rng.standard_normal(M * N))       # tiled layout, i.i.d. N(0,1)
    A0 = torch.from_numpy(A_host).to(dev)
    A = torch.empty_like(A0)
    T = torch.zeros(tq.t_size(M, N, NB, IB), dtype=torch.float64, device=dev)

    def factor_all(times):
        with torch.cuda.stream(stream):
            for ti, (tree, bs, fam) in enumerate(CASES):
                A.copy_(A0)                      # restore input; the 128 MB copy also flushes L2
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                tq.tiled_qr(A, M, N, NB, IB, tree, bs, fam, T=T, stream=stream)
                e1.record(stream)
                times.append((ti, e0, e1))

    # plans are built on first use (host), outside the timed region
    for _ in range(args.warmup):
        factor_all([])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = []
    with Clocks(local_rank) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for _ in range(args.steps):
            factor_all(ev)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches_per = tq.last_launch_count()
    per_tree = np.zeros(len(CASES))
    for ti, e0, e1 in ev:
        per_tree[ti] += e0.elapsed_time(e1)
    dev_ms = float(per_tree.sum())                       # device time of all factorizations
    t = torch.tensor([dev_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    ms_per_step = max_ms / args.steps
    total_flops = FLOPS * len(CASES) * args.steps * world
    value = total_flops / (max_ms / 1e3) / 1e9

    # end to end through the public API on host buffers (pinned): every factorization
    # uploads A, factors, and downloads A (R and V) and T; tiled_qr_host_async pipelines
    # the copies of consecutive calls with the neighbouring factorizations
    pin_A = torch.empty(M * N, dtype=torch.float64, pin_memory=True)
    pin_A.numpy()[:] = A_host
    outs = [(torch.empty(M * N, dtype=torch.float64, pin_memory=True),
             torch.empty(tq.t_size(M, N, NB, IB), dtype=torch.float64, pin_memory=True)) for _ in range(2)]
    e2e_steps = max(1, min(args.steps, 3))

    def e2e_run(nsteps):
        c = 0
        for _ in range(nsteps):
            for (tree, bs, fam) in CASES:
                R_o, T_o = outs[c & 1]
                tq.tiled_qr_host_async(pin_A.numpy(), R_o.numpy(), T_o.numpy(), M, N, NB, IB, tree, bs, fam,
                                       stream=stream)
                c += 1
        tq.host_wait()

    e2e_run(1)                                             # warm-up (plans, scratch)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    e2e_run(e2e_steps)
    e1.record(stream)
    e1.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = FLOPS * len(CASES) * e2e_steps * world / (float(t.item()) / 1e3) / 1e9
    h2d = M * N * 8 * len(CASES)
    d2h = (M * N + tq.t_size(M, N, NB, IB)) * 8 * len(CASES)

    if rank != 0:
        return
    peak, peak_src = fp64_peak()
    avg_launch_ms = dev_ms / (args.steps * len(CASES))
    achieved = FLOPS / (avg_launch_ms / 1e3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "m": M, "n": N, "nb": NB, "ib": IB, "p": P, "q": Q,
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "l2": "input restored by a 128 MB device copy before every factorization (outside the "
                         "events; flushes L2); the matrix itself (128 MB) exceeds L2",
                   "timing": "CUDA events around each tiled_qr launch on its stream, summed; max over ranks"},
        "per_tree_gflops": {f"{t}:{b} {f}": FLOPS * args.steps / (ms / 1e3) / 1e9
                            for (t, b, f), ms in zip(CASES, per_tree)},
        "fp64_peak_frac": achieved / peak,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": ncu_traffic(), "kernel": "tqr_persistent",
                     "peak_source": peak_src,
                     "flops_per_launch": FLOPS, "avg_launch_ms": avg_launch_ms},
        "clocks": clk.summary(),
        "e2e": {"value": e2e_value, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "tiled_qr_host_async (pinned host buffers; per factorization H2D A, factor, D2H A and T; "
                       "copies pipelined with neighbouring factorizations; CUDA events incl. the final wait)"},
        "gpu_launches": launches_per * len(CASES) * args.steps,
    }
    if not args.no_cpu_baseline and world == 1:
        budget = float(os.environ.get("TQR_CPU_BUDGET_S", "15"))
        g, fl, nt, tot, thr, el = oracle_sample(budget)
        line["cpu_baseline"] = {"value": g, "unit": "GFLOP/s", "cores": thr, "kind": "oracle",
                                "sample": f"first {nt} of {tot} tasks of the Greedy TT factorization of configs[1] "
                                          f"({el:.1f} s, oracle/numeric.py numpy fp64 kernels)"}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# configs[3]: tall-skinny, tile rows split across ranks, binary TT merge over NCCL
# ---------------------------------------------------------------------------
TALL = dict(p=2048, q=16, nb=256, ib=32)


def run_tall(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_1104_4475_b200 as tq
    from paper_1104_4475_b200 import dist as tdist

    p = args.tall_p or TALL["p"]
    q, nb, ib = TALL["q"], TALL["nb"], TALL["ib"]
    tree = args.tree
    m, n = p * nb, q * nb
    flops = 2.0 * n * n * (m - n / 3.0)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    r0, r1 = tdist.domain(p, world, rank)
    p_loc = r1 - r0
    g = torch.Generator(device=dev).manual_seed(SEED + 7919 * rank)
    A0 = torch.randn(p_loc * q * nb * nb, dtype=torch.float64, device=dev, generator=g)   # i.i.d. N(0,1)
    A = torch.empty_like(A0)
    stream = torch.cuda.current_stream()

    def one(times):
        A.copy_(A0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tdist.tall_skinny_qr(A, p, q, nb, ib, tree, 1, "TT")
        e1.record(stream)
        times.append((e0, e1))

    for _ in range(args.warmup):
        one([])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = []
    with Clocks(local_rank) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for _ in range(args.steps):
            one(ev)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = sum(e0.elapsed_time(e1) for e0, e1 in ev)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    value = flops * args.steps / (max_ms / 1e3) / 1e9
    if rank != 0:
        return
    peak, peak_src = fp64_peak()
    print(json.dumps({
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"configs[3]: tall-skinny fp64 tiled QR {m}x{n} (p={p} x q={q} tiles, nb={nb}, "
                               f"ib={ib}), i.i.d. N(0,1), tile-row domains per GPU reduced locally by {tree}, "
                               f"then a binary TT merge of the q x q R factors across GPUs (NCCL send/recv)",
                   "parallelism": f"tile-row domains x{world}",
                   "l2": "inputs (17 GB at full size) far exceed L2; restored by a device copy outside the events",
                   "timing": "CUDA events around tall_skinny_qr per rank (local factor + merges + NCCL), max over ranks"},
        "fp64_peak_frac": value / 1e3 / (peak * world),
        "roofline": {"bound": "tensor", "achieved": value / 1e3 / world, "peak": peak, "unit": "TFLOP/s",
                     "frac": value / 1e3 / world / peak, "traffic": None, "kernel": "tqr_persistent",
                     "peak_source": peak_src},
        "clocks": clk.summary(),
        "e2e": None,
        "gpu_launches": (1 + len(tdist.merge_schedule(world))) * args.steps,
    }), flush=True)


# ---------------------------------------------------------------------------
# configs[4]: q-sweep at fixed height p = 40, nb = 200 (the paper's experiment
# grid, §4), every tree, TT and TS kernels; one JSON line with
# the per-(q, tree, family) GFLOP/s table (a report, not the bench headline)
# ---------------------------------------------------------------------------
def run_qsweep(args, local_rank):
    import torch
    import paper_1104_4475_b200 as tq

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    p, nb, ib = 40, 200, 32
    qs = [1, 2, 4, 8, 16, 24, 32, 40]
    trees = [("flat", 1), ("fibonacci", 1), ("greedy", 1), ("asap", 1), ("plasma", 1), ("plasma", 5),
             ("plasma", 10), ("plasma", 20)]
    g = torch.Generator(device=dev).manual_seed(SEED)
    table = {}
    for q in qs:
        m, n = p * nb, q * nb
        flops = 2.0 * n * n * (m - n / 3.0)
        A0 = torch.randn(m * n, dtype=torch.float64, device=dev, generator=g)
        A = torch.empty_like(A0)
        T = torch.zeros(tq.t_size(m, n, nb, ib), dtype=torch.float64, device=dev)
        for fam in ("TT", "TS"):
            for (tree, bs) in trees:
                if tree == "asap" and fam == "TS":
                    continue
                best = None
                for it in range(2 + max(1, args.steps)):
                    A.copy_(A0)
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    tq.tiled_qr(A, m, n, nb, ib, tree, bs if tree != "asap" else q, fam, T=T)
                    e1.record()
                    e1.synchronize()
                    if it >= 2:
                        ms = e0.elapsed_time(e1)
                        best = ms if best is None else min(best, ms)
                table[f"q={q} {tree}:{bs} {fam}"] = round(flops / (best / 1e3) / 1e9, 1)
        del A0, A, T
    print(json.dumps({"workload": "configs[4]: q-sweep p=40, nb=200, ib=32, i.i.d. N(0,1); GFLOP/s, best of "
                                  f"{max(1, args.steps)} timed runs (CUDA events) per case",
                      "unit": "GFLOP/s", "gflops": table}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="square", choices=["square", "tall", "qsweep"],
                    help="square = configs[1] (default); tall = configs[3] partitioned over the ranks; "
                         "qsweep = configs[4] table (1 GPU)")
    ap.add_argument("--tree", default="greedy", help="tree of the local factorizations (tall workload)")
    ap.add_argument("--tall-p", type=int, default=0, help="override p of the tall workload (testing)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.workload == "qsweep":
        if rank == 0:
            run_qsweep(args, local_rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.workload == "tall":
            run_tall(args, rank, world, local_rank)
        else:
            run_gpu(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
