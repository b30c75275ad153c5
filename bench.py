"""Benchmark of the B200 tiled QR hot path (BASELINE.json metric).

Default (N = 1): configs[2], the paper's square grid point p = q = 40 tiles of
nb = 200 (8000 x 8000 fp64, i.i.d. N(0,1), ib = 32; §4 lines
1027-1031). A step = one tiled QR factorization with EACH of the trees
configs[2] names — Greedy, Fibonacci, FlatTree (Sameh-Kuck) — and each kernel
family (TT and TS, Algorithms 3 and 2): 6 factorizations.
value = 2n^2(m-n/3) flops x 6 / device time (GFLOP/s). The same line carries
configs[3] on one GPU (`tall_1gpu`: 524288 x 4096, nb = 256, Greedy with TS kernels, `--family`;
it also lists the same factorization by tree and kernel family).

N > 1 (`--gpus N`; relaunches itself under torch.distributed.run when
WORLD_SIZE is unset): configs[3] partitioned — contiguous tile-row domains per
GPU factored locally, then the binary TT merge of the q x q R factors over
NCCL (strong scaling: the total matrix is fixed).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
                    [--workload square|cfg1|tall|qsweep]
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

IB = 32
METRIC = "tiled QR fp64 GFLOP/s (2n²(m−n/3)) and % of B200 FP64 tensor peak, 1/2/4/8 GPU"
SEED = 2024
FAMILIES = ("TT", "TS")          # north_star: "executed with TT (triangle-on-triangle) and TS tile kernels"

# configs[2] (default) and configs[1] (--workload cfg1)
SQUARE = {
    "square": dict(p=40, q=40, nb=200, trees=[("greedy", 1), ("fibonacci", 1), ("flat", 1)],
                   name="configs[2]: fp64 square tiled QR 8000x8000 (p=q=40 tiles, nb=200, ib=32), i.i.d. N(0,1), "
                        "Greedy vs Fibonacci vs flat (Sameh-Kuck) tree, each with TT and with TS kernels"),
    "cfg1": dict(p=40, q=10, nb=200, trees=[("flat", 1), ("fibonacci", 1), ("greedy", 1), ("plasma", 1),
                                            ("plasma", 5), ("plasma", 10), ("plasma", 20)],
                 name="configs[1]: fp64 tiled QR 8000x2000 (p=40 x q=10 tiles, nb=200, ib=32), i.i.d. N(0,1), "
                      "each tree in turn (flat, fibonacci, greedy, plasma BS=1,5,10,20) with TT and with TS kernels"),
}
TALL = dict(p=2048, q=16, nb=256)

# PAPER.md §4 (lines 1017-1025, Table 7): the paper's own
# multicore numbers, quoted as context (other hardware, complex arithmetic).
PAPER_CONTEXT = {
    "hardware": "4 x 12-core AMD Opteron 8439 SE (48 cores, 2.8 GHz), theoretical peak 537.6 GFLOP/s "
                "(PAPER.md lines 1017-1025), PLASMA 2.3.1, nb=200, ib=32, p=40",
    "table7_greedy_gflops": {"q=10": 153.5, "q=40": 184.5},
    "note": "complex double arithmetic on CPUs; context only, not a target (vs_baseline stays null)",
}
TARGET_FRAC = 0.45   # stated target: achieved fraction of the FP64 tensor peak for the headline kernel


def flops_qr(m, n):
    return 2.0 * n * n * (m - n / 3.0)


def fp64_peak():
    """FP64 tensor peak = measured bf16 burst peak x the guide's nominal FP64/bf16 ratio (45/2250)."""
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return (mp["bf16_tflops"] * 45.0 / 2250.0,
                "of measured: MEASURED_PEAKS.json bf16_tflops x 45/2250 (guide nominal FP64/bf16 ratio)")
    except Exception:
        return 1590.0 * 45.0 / 2250.0, "of fallback: 1.59 PFLOP/s bf16 x 45/2250 (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler running during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, idx):
        self.idx = idx
        self.p = None
        self.out = ""

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
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
        for line in (self.out or "").strip().splitlines():
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


def ncu_traffic(workload):
    """Per-launch DRAM bytes of tqr_persistent from the committed ncu --set full summary of this workload."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", f"ncu_full_summary_{workload}.json")))
        return d.get("dram_bytes_per_launch"), d.get("command")
    except Exception:
        return None, None


# ---------------------------------------------------------------------------
# CPU oracle legs (cpu_baseline and --impl reference): the oracle as it stands
# ---------------------------------------------------------------------------
def oracle_sample(budget_s, p, q, nb, seed=SEED):
    """Run the oracle's tiled QR of the Greedy TT factorization of a p x q tile
    matrix task by task (oracle/numeric.py kernels in dag.expand order) until
    `budget_s` seconds have passed; return (GFLOP/s, flops, tasks done, tasks, threads, seconds)."""
    import qrinputs
    from oracle import dag, numeric as nu, schemes
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        threads = 1
    A = qrinputs.gaussian(p * nb, q * nb, seed)
    F = nu.Factor(np.array(A, order="F"), p, q, nb, IB, dag.expand(schemes.elim_list("greedy", p, q), p, q, "TT"))
    unit = nb ** 3 / 3.0
    done_flops, ntask = 0.0, 0
    t0 = time.perf_counter()
    for t in F.tasks:
        if t.kind == "GEQRT":
            taus, _ = nu.geqrt(F.tile(t.i, t.k), IB)
            F.tau[(0, t.i, t.k)] = taus
        elif t.kind == "UNMQR":
            nu.unmqr(F.tile(t.i, t.k), F.tau[(0, t.i, t.k)], F.tile(t.i, t.j))
        elif t.kind == "TTQRT":
            taus, _ = nu.ttqrt(F.tile(t.piv, t.k), F.tile(t.i, t.k), IB)
            F.tau[(1, t.i, t.k)] = taus
        else:
            nu.ttmqr(F.tile(t.i, t.k), F.tau[(1, t.i, t.k)], F.tile(t.piv, t.j), F.tile(t.i, t.j))
        done_flops += t.weight * unit
        ntask += 1
        if time.perf_counter() - t0 > budget_s:
            break
    el = time.perf_counter() - t0
    return done_flops / el / 1e9, done_flops, ntask, len(F.tasks), threads, el


def workload_of(args, world):
    if args.workload == "auto":
        return "tall" if world > 1 else "square"
    return args.workload


def run_reference(args, rank, world):
    """--impl reference: no reference implementation exists (the reference mount
    holds only the paper); the oracle is timed as it stands on the host cores, each
    step a bounded sample of the same workload's Greedy TT factorization."""
    if rank != 0:
        return
    wl = workload_of(args, world)
    if wl == "tall":
        p, q, nb = TALL["p"] // 64, TALL["q"], TALL["nb"]     # sample: the leading 32 tile rows' domain
        name = (f"configs[3]: tall-skinny fp64 tiled QR {TALL['p'] * nb}x{TALL['q'] * nb} (p={TALL['p']} x "
                f"q={TALL['q']} tiles, nb={nb}, ib={IB}), i.i.d. N(0,1), partitioned over {world} GPU(s)")
    else:
        c = SQUARE[wl if wl in SQUARE else "square"]
        p, q, nb, name = c["p"], c["q"], c["nb"], c["name"]
    budget = float(os.environ.get("TQR_REF_BUDGET_S", "8"))
    vals, last = [], None
    for _ in range(args.warmup):
        oracle_sample(min(budget, 2.0), p, q, nb)
    for _ in range(args.steps):
        last = oracle_sample(budget, p, q, nb)
        vals.append(last[0])
    v = float(np.mean(vals))
    g, fl, nt, tot, thr, el = last
    sample = (f"first {nt} of {tot} tasks (in list order) of the Greedy TT factorization of a {p}x{q}-tile "
              f"nb={nb} matrix, {budget:g} s budget per step, oracle/numeric.py kernels (numpy fp64)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": budget * 1000.0, "higher_is_better": True,
        "scaling": "strong" if wl == "tall" else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": name, "sample": sample},
        "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": thr, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
# GPU leg: square workloads (configs[2] default, configs[1])
# ---------------------------------------------------------------------------
def run_square(args, rank, world, local_rank, wl):
    import torch
    import torch.distributed as dist
    import paper_1104_4475_b200 as tq

    c = SQUARE[wl]
    P, Q, NB = c["p"], c["q"], c["nb"]
    M, N = P * NB, Q * NB
    FLOPS = flops_qr(M, N)
    cases = [(t, b, f) for f in FAMILIES for (t, b) in c["trees"]]
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
            for ti, (tree, bs, fam) in enumerate(cases):
                A.copy_(A0)                      # restore input; the copy (>= 128 MB) also flushes L2
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                tq.tiled_qr(A, M, N, NB, IB, tree, bs, fam, T=T, stream=stream)
                e1.record(stream)
                times.append((ti, e0, e1))

    for _ in range(args.warmup):             # plans are built on first use (host), outside the timed region
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
    per_case = np.zeros(len(cases))
    for ti, e0, e1 in ev:
        per_case[ti] += e0.elapsed_time(e1)
    dev_ms = float(per_case.sum())
    t = torch.tensor([dev_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    value = FLOPS * len(cases) * args.steps * world / (max_ms / 1e3) / 1e9

    # end to end through the public API on pinned host buffers: every factorization uploads
    # A, factors, and downloads A (R and V) and T; tiled_qr_host_async pipelines consecutive calls
    pin_A = torch.empty(M * N, dtype=torch.float64, pin_memory=True)
    pin_A.numpy()[:] = A_host
    outs = [(torch.empty(M * N, dtype=torch.float64, pin_memory=True),
             torch.empty(tq.t_size(M, N, NB, IB), dtype=torch.float64, pin_memory=True)) for _ in range(2)]
    e2e_steps = max(1, min(args.steps, 3))

    def e2e_run(nsteps):
        k = 0
        for _ in range(nsteps):
            for (tree, bs, fam) in cases:
                R_o, T_o = outs[k & 1]
                tq.tiled_qr_host_async(pin_A.numpy(), R_o.numpy(), T_o.numpy(), M, N, NB, IB, tree, bs, fam,
                                       stream=stream)
                k += 1
        tq.host_wait()

    e2e_run(1)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    e2e_run(e2e_steps)
    e1.record(stream)
    e1.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = FLOPS * len(cases) * e2e_steps * world / (float(t.item()) / 1e3) / 1e9
    h2d = M * N * 8 * len(cases)
    d2h = (M * N + tq.t_size(M, N, NB, IB)) * 8 * len(cases)
    del pin_A, outs

    tall = None
    if world == 1 and wl == "square" and not args.no_tall:
        del A0, A, T
        torch.cuda.empty_cache()
        tall = run_tall(args, 0, 1, local_rank, nested=True)

    if rank != 0:
        return
    peak, peak_src = fp64_peak()
    avg_launch_ms = dev_ms / (args.steps * len(cases))
    achieved = FLOPS / (avg_launch_ms / 1e3) / 1e12
    traffic, traffic_cmd = ncu_traffic(wl)
    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": c["name"], "m": M, "n": N, "nb": NB, "ib": IB, "p": P, "q": Q,
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "l2": f"input restored by a {M * N * 8 >> 20} MB device copy before every factorization "
                         "(outside the events; flushes L2); the matrix itself exceeds L2",
                   "timing": "CUDA events around each tiled_qr launch on its stream, summed; max over ranks"},
        "per_case_gflops": {f"{tr}:{b} {f}": FLOPS * args.steps / (ms / 1e3) / 1e9
                            for (tr, b, f), ms in zip(cases, per_case)},
        "fp64_peak_frac": achieved / peak,
        "target_frac": TARGET_FRAC,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_cmd,
                     "kernel": "tqr_persistent", "peak_source": peak_src,
                     "flops_per_launch": FLOPS, "avg_launch_ms": avg_launch_ms},
        "clocks": clk.summary(),
        "e2e": {"value": e2e_value, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "api": "tiled_qr_host_async (pinned host buffers; per factorization H2D A, factor, D2H A and T; "
                       "copies pipelined with neighbouring factorizations; CUDA events incl. the final wait)"},
        "gpu_launches": launches_per * len(cases) * args.steps,
        "paper_context": PAPER_CONTEXT,
    }
    if tall is not None:
        line["tall_1gpu"] = tall
    if not args.no_cpu_baseline and world == 1:
        budget = float(os.environ.get("TQR_CPU_BUDGET_S", "15"))
        g, fl, nt, tot, thr, el = oracle_sample(budget, P, Q, NB)
        line["cpu_baseline"] = {"value": g, "unit": "GFLOP/s", "cores": thr, "kind": "oracle",
                                "sample": f"first {nt} of {tot} tasks of the Greedy TT factorization of the same "
                                          f"{M}x{N} matrix ({el:.1f} s, oracle/numeric.py numpy fp64 kernels)"}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# configs[3]: tall-skinny, tile rows split across ranks, binary TT merge over NCCL
# ---------------------------------------------------------------------------
def run_tall(args, rank, world, local_rank, nested=False):
    import torch
    import torch.distributed as dist
    import paper_1104_4475_b200 as tq
    from paper_1104_4475_b200 import dist as tdist

    p = args.tall_p or TALL["p"]
    q, nb = TALL["q"], TALL["nb"]
    tree, fam = args.tree, args.family
    m, n = p * nb, q * nb
    flops = flops_qr(m, n)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    r0, r1 = tdist.domain(p, world, rank)
    p_loc = r1 - r0
    g = torch.Generator(device=dev).manual_seed(SEED + 7919 * rank)
    A0 = torch.randn(p_loc * q * nb * nb, dtype=torch.float64, device=dev, generator=g)   # i.i.d. N(0,1)
    A = torch.empty_like(A0)
    stream = torch.cuda.current_stream()
    steps = args.tall_steps if nested else args.steps
    warm = 1 if nested else args.warmup
    launches = [0]

    def one(times):
        A.copy_(A0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tdist.tall_skinny_qr(A, p, q, nb, IB, tree, 1, fam)
        e1.record(stream)
        times.append((e0, e1))

    for _ in range(warm):
        one([])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = []
    with Clocks(local_rank) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for _ in range(steps):
            one(ev)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = sum(e0.elapsed_time(e1) for e0, e1 in ev)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    value = flops * steps / (max_ms / 1e3) / 1e9
    merges = sum(1 for pairs in tdist.merge_schedule(world) for (d, s) in pairs if d == rank)

    # end to end (N > 1 only; at N = 1 the nested object is a device-timed companion line): every
    # step uploads this rank's domain from pinned host memory, factors, and reads R back on rank 0
    e2e = None
    if not nested:
        pin = torch.empty(A0.numel(), dtype=torch.float64, pin_memory=True)
        pin.copy_(A0)
        r_host = torch.empty(q * q * nb * nb, dtype=torch.float64, pin_memory=True)

        def e2e_step():
            A.copy_(pin, non_blocking=True)
            F = tdist.tall_skinny_qr(A, p, q, nb, IB, tree, 1, fam)
            if F.R is not None:
                r_host.copy_(F.R, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            e2e_step()
        e1.record(stream)
        e1.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = {"value": flops * steps / (float(t.item()) / 1e3) / 1e9, "unit": "GFLOP/s",
               "h2d_bytes_per_step": p * q * nb * nb * 8, "d2h_bytes_per_step": q * q * nb * nb * 8,
               "api": "tall_skinny_qr on each rank: H2D of the rank's domain from pinned memory, local tiled_qr, "
                      "NCCL merges, D2H of R on rank 0; CUDA events, max over ranks"}
        del pin, r_host
    peak, peak_src = fp64_peak()
    out = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": steps,
        "warmup": warm, "ms_per_step": max_ms / steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"configs[3]: tall-skinny fp64 tiled QR {m}x{n} (p={p} x q={q} tiles, nb={nb}, "
                               f"ib={IB}), i.i.d. N(0,1), tile-row domains per GPU reduced locally by {tree} "
                               f"with {fam} kernels, then a binary TT merge of the q x q R factors across GPUs "
                               f"(NCCL send/recv)",
                   "tree": tree, "family": fam,
                   "parallelism": f"tile-row domains x{world}",
                   "l2": "inputs (17 GB at full size) far exceed L2; restored by a device copy outside the events",
                   "timing": "CUDA events around tall_skinny_qr per rank (local factor + merges + NCCL), max over ranks"},
        "fp64_peak_frac": value / 1e3 / (peak * world),
        "roofline": {"bound": "tensor", "achieved": value / 1e3 / world, "peak": peak, "unit": "TFLOP/s",
                     "frac": value / 1e3 / world / peak, "traffic": ncu_traffic("tall")[0], "kernel": "tqr_persistent",
                     "peak_source": peak_src},
        "clocks": clk.summary(),
        "e2e": e2e,
        "gpu_launches": (1 + merges) * steps,
    }
    if nested and world == 1 and not args.tall_p:
        # the same 1-GPU factorization by tree and kernel family (one warm-up, one timed run each):
        # TS kernels on full tiles keep the tensor pipe busier
        by = {}
        T = torch.empty(tq.t_size(m, n, nb, IB), dtype=torch.float64, device=dev)
        for tr, bs, fm in (("greedy", 1, "TT"), ("greedy", 1, "TS"), ("flat", 1, "TS"), ("plasma", 64, "TS")):
            ts = []
            for _ in range(2):
                A.copy_(A0)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                tq.tiled_qr(A, m, n, nb, IB, tr, bs, fm, T=T)
                e1.record(stream)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            by[f"{tr}:{bs} {fm}"] = flops / (ts[-1] / 1e3) / 1e9
        out["local_by_tree_gflops"] = by
        del T
    del A0, A
    torch.cuda.empty_cache()
    if nested:
        return out
    if rank == 0:
        out["paper_context"] = PAPER_CONTEXT
        out["nccl"] = {"world": world, "backend": dist.get_backend() if world > 1 else None,
                       "version": ".".join(map(str, torch.cuda.nccl.version())) if world > 1 else None}
        print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------
# configs[4]: q-sweep at fixed height p = 40, nb = 200 (the paper's experiment
# grid, §4), every tree, TT and TS kernels; one JSON line with
# the per-(q, tree, family) GFLOP/s table (mean over the timed runs)
# ---------------------------------------------------------------------------
def run_qsweep(args, local_rank):
    import torch
    import paper_1104_4475_b200 as tq

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    p, nb = 40, 200
    qs = [1, 2, 4, 8, 16, 24, 32, 40]
    trees = [("flat", 1), ("fibonacci", 1), ("greedy", 1), ("asap", 1), ("plasma", 1), ("plasma", 5),
             ("plasma", 10), ("plasma", 20)]
    g = torch.Generator(device=dev).manual_seed(SEED)
    table = {}
    nrun = max(1, args.steps)
    for q in qs:
        m, n = p * nb, q * nb
        flops = flops_qr(m, n)
        A0 = torch.randn(m * n, dtype=torch.float64, device=dev, generator=g)
        A = torch.empty_like(A0)
        T = torch.zeros(tq.t_size(m, n, nb, IB), dtype=torch.float64, device=dev)
        for fam in FAMILIES:
            for (tree, bs) in trees:
                if tree == "asap" and fam == "TS":
                    continue
                tot = 0.0
                for it in range(2 + nrun):
                    A.copy_(A0)
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    tq.tiled_qr(A, m, n, nb, IB, tree, bs if tree != "asap" else q, fam, T=T)
                    e1.record()
                    e1.synchronize()
                    if it >= 2:
                        tot += e0.elapsed_time(e1)
                table[f"q={q} {tree}:{bs} {fam}"] = round(flops * nrun / (tot / 1e3) / 1e9, 1)
        del A0, A, T
    print(json.dumps({"workload": "configs[4]: q-sweep p=40, nb=200, ib=32, i.i.d. N(0,1); GFLOP/s, mean over "
                                  f"{nrun} timed runs (CUDA events; 2 warm-up runs) per case",
                      "unit": "GFLOP/s", "gflops": table}), flush=True)


def self_launch(args):
    """--gpus N > 1 without a torchrun environment: relaunch under torch.distributed.run."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tall", action="store_true", help="skip the nested configs[3] 1-GPU measurement")
    ap.add_argument("--tall-steps", type=int, default=2, help="timed steps of the nested configs[3] measurement")
    ap.add_argument("--workload", default="auto", choices=["auto", "square", "cfg1", "tall", "qsweep"],
                    help="auto = configs[2] at N=1, configs[3] partitioned at N>1; cfg1 = configs[1]; "
                         "qsweep = configs[4] table (1 GPU)")
    ap.add_argument("--tree", default="greedy", help="tree of the local factorizations (tall workload)")
    ap.add_argument("--family", default="TS", choices=["TT", "TS"],
                    help="kernel family of the local factorizations (tall workload; the merge is TT)")
    ap.add_argument("--tall-p", type=int, default=0, help="override p of the tall workload (testing)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    wl = workload_of(args, world)
    if wl == "qsweep":
        if rank == 0:
            run_qsweep(args, local_rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if wl == "tall":
            run_tall(args, rank, world, local_rank)
        else:
            run_square(args, rank, world, local_rank, wl)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
