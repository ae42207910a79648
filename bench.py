"""Benchmark of the butterfly apply hot path on B200 (BASELINE.json metric:
complex samples/s = N * nRHS / t_apply, plus % of HBM roofline).

Default workload: BASELINE config 2 — FIO geometry N=2^20, r=16, leaf 16
(L=16), complex128, 1 RHS — the single-GPU config the north star's ">= 60% of
HBM roofline at N >= 2^20" target is quoted on. Factors are a seeded
synthetic chain at the reference's exact shapes (full CPU construction of
config 2 takes ~10-19 h in the reference).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config cfg2|cfg1|cfg0] [--dtype c128|c64] [--rhs k]

--impl reference times the reference algorithm's CPU path (the NumPy oracle
port in oracle/, the reference itself being pure Python that cannot travel
to the GPU box) on the same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (kernel, n, r, leaf, default rhs); 2-D (radon) configs give the grid side
    # as leaf = leaf box side and n = n_side^2 (quadtree over Morton-ordered points)
    "cfg0": ("fio", 1 << 10, 12, 8, 1),
    "cfg1": ("dftp", 1 << 16, 8, 16, 64),
    "cfg2": ("fio", 1 << 20, 16, 16, 1),
    "cfg3": ("radon2d", 1 << 16, 25, 4, 16),
    "cfg4a": ("fio", 1 << 24, 16, 16, 64),
    "cfg4b": ("radon2d", 1 << 20, 25, 4, 16),
}


def partition_for(kern, n, leaf):
    import paper_1502_01379_b200 as bf
    if kern == "radon2d":
        return bf.make_quadtree_partition(int(round(n ** 0.5)), leaf)
    return bf.make_partition(n, leaf)
METRIC = "BF apply complex-samples/s (N*nRHS/s)"
FACTOR_SEED = 20240801   # the reference's conftest seed (pkg/tests/conftest.py:42-44)


def bench_config(name, kern, n, r, leaf, k, p, dtype, world=1, parallelism=None):
    """The `config` object of both arms' JSON lines (identical keys and values)."""
    return {"workload": f"{name} {kern.upper()} N={n} r={r} leaf={leaf} (L={p.levels}) k={k} {dtype}, "
                        f"synthetic seeded factors (bench_chain seed {FACTOR_SEED})",
            "n": n, "rank": r, "levels": p.levels, "rhs": k, "parallelism": parallelism or f"replicas{world}",
            "l2": l2_note(chain_bytes(p, r, 16 if dtype == "c128" else 8))}


def l2_note(nbytes):
    if nbytes > 126e6:
        return f"inputs larger than L2: each step streams the whole factor chain ({nbytes / 1e9:.2f} GB; L2 126 MB)"
    return (f"factor chain ({nbytes / 1e6:.1f} MB) fits the 126 MB L2 and stays resident between steps "
            "(a latency-bound workload; no flush)")


def chain_bytes(p, r, esz):
    import paper_1502_01379_b200 as bf
    shapes, leaf_shape = bf.level_geometry(p, r)
    elems = 2 * int(np.prod(leaf_shape)) + 2 * sum(int(np.prod(s)) for _, _, s in shapes)
    return esz * elems + (esz // 2) * p.mid_nodes ** 2 * r


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--dtype", default="c128", choices=["c128", "c64"])
    ap.add_argument("--rhs", type=int, default=0, help="right-hand sides (default: the config's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="use the node-sharded path even at one rank")
    ap.add_argument("--no-also", action="store_true", help="skip the companion configs[1] measurement")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = each GPU keeps the config's per-GPU size (N = n x GPUs, 1-D "
                         "configs), strong = the config's N split over the GPUs")
    ap.add_argument("--exchange", default="push", choices=["push", "nccl"],
                    help="N>1 middle exchange: fused peer stores (symmetric memory) or pack + NCCL all-to-all")
    return ap.parse_args()


def algorithmic(f, k, esz):
    """Compulsory bytes/flops of one apply:
    bytes = esz*(nnz - nnz_M) + esz/2*nnz_M + 2*esz*N*k ; flops = 8k(nnz - nnz_M) + 2k nnz_M."""
    rep = f.nnz_report()
    nnz, nm = rep.total, rep.middle
    return esz * (nnz - nm) + esz // 2 * nm + 2 * esz * f.n * k, 8 * k * (nnz - nm) + 2 * k * nm


def launch_flops(f, k, folded=False):
    """Algorithmic flops of each launch of the forward chain (8 per complex multiply-add,
    2 per real-weight scaling of the fused middle factor), in launch order. folded: the leaf
    factors are folded into the outermost levels at plan upload (plan_fold_leaves), whose
    blocks are then n0 x C and whose launches replace the two leaf launches."""
    p = f.partition
    nb, n0, r = f.u_outer.blocks.shape
    out = [] if folded else [("V*", 8 * k * nb * n0 * r)]
    for tf in reversed(f.h_chain):
        fl = 8 * k * tf.nnz
        name = f"H{tf.level}*"
        if folded and tf.level == p.levels - 1:
            fl, name = 8 * k * (tf.nnz // r) * n0, name + " (V folded in)"
        out.append((name, fl + (2 * k * f.middle.nnz if tf.level == p.half else 0)))
    for tf in f.g_chain:
        fl, name = 8 * k * tf.nnz, f"G{tf.level}"
        if folded and tf.level == p.levels - 1:
            fl, name = 8 * k * (tf.nnz // r) * n0, name + " (U folded in)"
        out.append((name, fl))
    if not folded:
        out.append(("U", 8 * k * nb * n0 * r))
    return out


def launch_bytes(f, k, esz, folded=False):
    """Bytes of each launch of the forward chain, in launch order: factor bytes + input
    vector + output vector (M is fused into the last H* launch). folded: see launch_flops —
    the outermost levels read n0 x C blocks and the chain input / write the chain output."""
    p, r = f.partition, f.rank
    nb, n0, _ = f.u_outer.blocks.shape
    out = [] if folded else [("V*", esz * nb * n0 * r + esz * k * (nb * n0 + nb * r))]
    for tf in reversed(f.h_chain):
        rows, cols = tf.shape
        extra = (esz // 2) * f.middle.nnz if tf.level == p.half else 0
        if folded and tf.level == p.levels - 1:
            out.append((f"H{tf.level}* (V folded in)", esz * (tf.nnz // r) * n0 + esz * k * (nb * n0 + cols) + extra))
        else:
            out.append((f"H{tf.level}*", esz * tf.nnz + esz * k * (rows + cols) + extra))
    for tf in f.g_chain:
        rows, cols = tf.shape
        if folded and tf.level == p.levels - 1:
            out.append((f"G{tf.level} (U folded in)", esz * (tf.nnz // r) * n0 + esz * k * (nb * n0 + cols)))
        else:
            out.append((f"G{tf.level}", esz * tf.nnz + esz * k * (rows + cols)))
    if not folded:
        out.append(("U", esz * nb * n0 * r + esz * k * (nb * n0 + nb * r)))
    return out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.proc, self.path = index, None, None

    def start(self):
        try:
            self.path = f"/tmp/bf_clocks_{os.getpid()}.csv"
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6 and parts[0].isdigit():
                rows.append(parts)
        if not rows:
            return None
        sm = [int(r[0]) for r in rows]
        busy = [s for s in sm if s > 600] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(int(r[1]) for r in rows), "reasons": reasons,
                "samples": len(rows)}


def rhs_input(n, k, seed=0):
    """g = complex_normal with SeedSequence(seed, spawn_key=(4, 0)) as the reference bench (bench.py:208-213)."""
    rng = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(4, 0)))
    g = rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))
    return g


def oracle_chain(fh):
    from oracle import chain as ochain
    return ochain.Chain(fh.n, fh.partition.levels, fh.rank, fh.u_outer.blocks,
                        [(t.level, t.blocks) for t in fh.g_chain], fh.middle.weights,
                        [(t.level, t.blocks) for t in fh.h_chain], fh.v_outer.blocks)


def rel2(got, want):
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))


def time_cpu(fh, g, budget_s=20.0, max_steps=5):
    """The reference algorithm on host cores: oracle port of ButterflyFactors.apply (median of
    runs); also returns its output for the GPU result's relative error."""
    from oracle import chain as ochain
    oc = oracle_chain(fh)
    times = []
    t_start = time.perf_counter()
    while len(times) < max_steps and (not times or time.perf_counter() - t_start < budget_s):
        t0 = time.perf_counter()
        want = ochain.apply(oc, g)
        times.append(time.perf_counter() - t0)
    return statistics.median(times), len(times), want


def dev_time(fn, steps, warm):
    """ms per call of fn on the current stream: CUDA events around `steps` calls after `warm`."""
    import torch
    for _ in range(warm):
        fn()
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


LIVE_PEAKS = {}   # bf_measure_peaks in this process (measure_live_peaks)


def measure_live_peaks():
    """FP64 DMMA / DFMA peaks and streaming-read / copy bandwidth measured in this process on
    this GPU (bf_measure_peaks over an 8 GiB buffer: far larger than L2), the denominators of the
    FP64 and read-dominated rooflines; MEASURED_PEAKS.json has neither."""
    import torch

    from paper_1502_01379_b200 import _lib
    buf = torch.empty(8 << 30, dtype=torch.uint8, device="cuda")
    out = (ctypes.c_double * 4)()
    _lib.check(_lib.load().bf_measure_peaks(out, ctypes.c_void_p(buf.data_ptr()), buf.numel(),
                                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
               "bf_measure_peaks")
    del buf
    torch.cuda.empty_cache()
    LIVE_PEAKS.update(dmma_tflops=out[0], dfma_tflops=out[1], read_gbs=out[2], copy_gbs=out[3],
                      how="bf_measure_peaks: mma.sync m8n8k4 f64 loop, DFMA loop, __ldcs read stream over 8 GiB "
                          "and a 4 GiB device-to-device cudaMemcpyAsync; best of 5 after a warm-up, in this process")
    return dict(LIVE_PEAKS)


def _peaks():
    pk = {}
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")):
        pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    fp = json.load(open(os.path.join(ROOT, "profiles", "r01_fp64_peaks.json")))
    dmma = LIVE_PEAKS.get("dmma_tflops", float(fp["dmma_m8n8k4_tflops"]))
    read = LIVE_PEAKS.get("read_gbs", float(fp["read_gbs"]))
    return float(pk.get("hbm_gbs", 6550.0)), float(dmma), float(read)


def _rate(f, k, esz, ms):
    """Algorithmic rates of one apply: GB/s against the HBM peak when k < 8 (streaming levels),
    FP64 TF/s against the DMMA peak otherwise."""
    b, fl = algorithmic(f, k, esz)
    hbm, dmma, _ = _peaks()
    out = {"algorithmic_bytes": b, "algorithmic_flops": fl, "gbs": b / (ms / 1e3) / 1e9,
           "tflops": fl / (ms / 1e3) / 1e12}
    if k < 8:
        out.update(bound="hbm", frac=out["gbs"] / hbm, peak=hbm)
    elif esz == 16:
        # flops the tensor pipe executes: 6 per complex multiply-add instead of 8 (3-multiplication
        # form), and the leaf-folded outermost levels do n0 C instead of n0 r + r C per block
        nb, n0, r = f.u_outer.blocks.shape
        last = f.g_chain[-1].nnz if f.g_chain else 0
        executed = 0.75 * (fl - 8 * k * (2 * nb * n0 * r + 2 * last - 2 * (last // r) * n0))
        out.update(bound="fp64 tensor (DMMA)", frac=out["tflops"] / dmma, peak=dmma,
                   executed_tflops=executed / (ms / 1e3) / 1e12, executed_frac=executed / (ms / 1e3) / 1e12 / dmma,
                   note="tflops / frac count the reference factor list at 8 flops per complex multiply-add "
                        "(SURVEY 8(d)) and can exceed the pipe's peak; executed_* count what the DMMA pipe runs "
                        "(3 real products per complex one, leaf factors folded into the outermost levels)")
    else:
        out.update(bound="fp32 (FFMA)", frac=None, peak=None)
    return out


def companion_cfg(name, dtype, rhs, steps, warm, cols=1):
    """One BASELINE config on its own plan: device-timed apply (CUDA events, bf_apply graph
    replay), algorithmic rate, and the relative error of `cols` output columns against the
    oracle port on the identical factors and inputs."""
    import torch

    from paper_1502_01379_b200.synthetic import bench_chain
    kern, n, r, leaf, k0 = CONFIGS[name]
    k = rhs or k0
    esz = 16 if dtype == "c128" else 8
    p = partition_for(kern, n, leaf)
    fh = bench_chain(p, r, seed=FACTOR_SEED)
    plan = fh.plan(dtype)
    tdt = torch.complex128 if dtype == "c128" else torch.complex64
    g_host = rhs_input(n, k)
    g = torch.from_numpy(g_host).cuda().to(tdt)
    out = torch.empty_like(g)
    ws = torch.empty(plan.workspace_bytes(k), dtype=torch.uint8, device="cuda")
    nsteps = max(3, min(steps, 20))
    ms = dev_time(lambda: plan.apply(g, out=out, workspace=ws), nsteps, max(3, warm))
    graph_ms = None
    if ms < 0.1:
        # latency-bound chain: one host call per apply costs more than the device work, so
        # also time 50 applies captured into one CUDA graph (device time per apply)
        reps = 50
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg, capture_error_mode="thread_local"):
            for _ in range(reps):
                plan.apply(g, out=out, workspace=ws)
        graph_ms = dev_time(cg.replay, 5, 2) / reps
    t0 = time.perf_counter()
    plan.apply(g_host, out=np.empty_like(g_host, dtype=plan.np_dtype))     # host buffers (pageable)
    e2e_ms = (time.perf_counter() - t0) * 1e3
    from oracle import chain as ochain
    t1 = time.perf_counter()
    want = ochain.apply(oracle_chain(fh), g_host[:, :cols])
    t_cpu = time.perf_counter() - t1
    err = rel2(out[:, :cols].cpu().numpy().astype(np.complex128), want)
    res = {"workload": bench_config(name, kern, n, r, leaf, k, p, dtype)["workload"], "value": n * k / (ms / 1e3),
           "unit": "samples/s", "ms_per_step": ms, "steps": nsteps, "roofline": _rate(fh, k, esz, ms),
           "device_ms_per_apply_graph": graph_ms,
           "rel_err": {"value": err, "columns": cols, "tolerance": 1e-11 if dtype == "c128" else 1e-5},
           "e2e_ms_one_call_pageable": e2e_ms,
           "cpu_reference": {"value": n * cols / t_cpu, "unit": "samples/s", "ms": t_cpu * 1e3, "k": cols,
                             "kind": "port"}}
    del plan, g, out, ws
    return res


def companion_many_rhs(plan, f, n, steps, warm, k=256, cols=2):
    """BASELINE configs[2]'s 256-RHS complex128 apply on the same cfg2 plan: device time,
    algorithmic FP64 rate against the measured DMMA peak, and the relative error of `cols`
    output columns against the oracle port."""
    import torch
    g_host = rhs_input(n, k)
    g = torch.from_numpy(g_host).cuda()
    out = torch.empty_like(g)
    ws = torch.empty(plan.workspace_bytes(k), dtype=torch.uint8, device="cuda")
    nsteps = max(3, min(steps, 10))
    ms = dev_time(lambda: plan.apply(g, out=out, workspace=ws), nsteps, max(2, min(warm, 3)))
    from oracle import chain as ochain
    want = ochain.apply(oracle_chain(f), g_host[:, :cols])
    err = rel2(out[:, :cols].cpu().numpy(), want)
    del g, out, ws
    return {"workload": f"cfg2 k={k} c128 (same plan)", "value": n * k / (ms / 1e3), "unit": "samples/s",
            "ms_per_step": ms, "steps": nsteps, "roofline": _rate(f, k, 16, ms),
            "rel_err": {"value": err, "columns": cols, "tolerance": 1e-11}}


def companion_same_plan_c64(f, n, steps, warm, cols=1):
    """BASELINE configs[2]'s complex64 mode: the same cfg2 factors in a c64 plan, 1 RHS."""
    import torch
    plan = f.plan("c64")
    g_host = rhs_input(n, 1)
    g = torch.from_numpy(g_host).cuda().to(torch.complex64)
    out = torch.empty_like(g)
    ws = torch.empty(plan.workspace_bytes(1), dtype=torch.uint8, device="cuda")
    nsteps = max(5, min(steps, 20))
    ms = dev_time(lambda: plan.apply(g, out=out, workspace=ws), nsteps, max(3, warm))
    from oracle import chain as ochain
    want = ochain.apply(oracle_chain(f), g_host[:, :cols])
    err = rel2(out[:, :cols].cpu().numpy().astype(np.complex128), want)
    del plan, g, out, ws
    return {"workload": "cfg2 k=1 c64 (same factors, complex64 plan)", "value": n / (ms / 1e3),
            "unit": "samples/s", "ms_per_step": ms, "steps": nsteps, "roofline": _rate(f, 1, 8, ms),
            "rel_err": {"value": err, "columns": cols, "tolerance": 1e-5}}


def construction_flops(p, r, q=3, iters=3):
    """Algorithmic FP64 flops of one sampling-mode factorize (8 per complex multiply-add), an
    upper-bound model of the reference algorithm's arithmetic with the
    sample sets at their caps: per middle block (side s, |rows| = |cols| = r (q + 1), basis
    width t = 3 r) the sweep pivots' projections 2 (iters + 1) x r picks x |rows| s, the two
    Gram matrices |cols|^2 s, the two bases (CGS2) 2 t^2 s each, the assembly 2 s t r; per
    recursion level and stack (rows x 2r) a QR 2 rows w^2, a one-sided Jacobi SVD counted as
    10 sweeps x min(rows, w) w^2, and A V. cfg2: 58 TFLOP middle level + 110 TFLOP recursion."""
    m, s = p.mid_nodes, p.mid_side
    rs, t = r * (q + 1), 3 * r
    per_block = 8 * (2 * (iters + 1) * r * rs * s + 2 * rs * rs * s + 2 * 2 * t * t * s + 2 * s * t * r)
    mid = per_block * m * m
    # recursion (construct.py:127-163): per side m slabs of s rows; at level l a slab splits into
    # 2^l m / 2 x 2 stacks of s / 2^(l+1) rows x 2r columns (the entry count is level-invariant):
    # QR 2 rows w^2, one-sided Jacobi ~10 min(rows, w) w^2, the product A V rows w r
    rec, rows, w = 0, s, 2 * r
    for lvl in range(p.levels - p.half):
        n_stack = (s // rows) * m
        mrow = max(1, rows // 2)
        rec += 8 * n_stack * (2 * mrow * w * w + 10 * min(mrow, w) * w * w + mrow * w * r)
        rows = max(2, rows // 2)
    return mid + 2 * m * rec


def companion_construction(name, cpu_blocks=2):
    """BASELINE configs[2]'s construction, the reference bench's row (factorize time, eps_a,
    apply time; reference bench.py:202-222): full GPU `factorize` (sampling mode, FIO kernel,
    seed 0), eps_a on 256 sampled rows (bench.py:84-97), one apply of the built chain; the
    reference algorithm's CPU time extrapolated from sampled middle blocks and one slab
    recursion (the oracle port, bitwise equal to the reference on the pinned fixtures)."""
    import torch

    import paper_1502_01379_b200 as bf
    from paper_1502_01379_b200 import construct as bc
    kern, n, r, leaf, _ = CONFIGS[name]
    p = partition_for(kern, n, leaf)
    ker = bf.FioKernel(n) if kern == "fio" else bf.DftPlusKernel(n)
    bc.MiddleSampler(ker, p, r).blocks([(0, 0)])          # module load, first launches
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fb = bf.factorize(ker, p, r, seed=0)
    torch.cuda.synchronize()
    t_fac = time.perf_counter() - t0
    t1 = time.perf_counter()
    eps = bf.estimate_eps_a(fb, bf.RowSampledReference(ker), 256, np.random.SeedSequence(0, spawn_key=(4, 0)))
    t_eps = time.perf_counter() - t1
    import torch as _t
    plan = fb.plan("c128")
    g = _t.from_numpy(rhs_input(n, 1)).cuda()
    out = _t.empty_like(g)
    ws = _t.empty(plan.workspace_bytes(1), dtype=_t.uint8, device="cuda")
    ms = dev_time(lambda: plan.apply(g, out=out, workspace=ws), 10, 3)
    del plan, fb, g, out, ws
    # CPU: the reference algorithm on sampled middle blocks + one slab recursion, extrapolated
    from oracle import construct as ocons
    from oracle import entries as oent
    from oracle import lowrank as olr
    m, side = p.mid_nodes, p.mid_side
    ent = oent.EntryOracle(kern, n)
    rng = np.random.default_rng(0)
    picks = [(int(rng.integers(m)), int(rng.integers(m))) for _ in range(cpu_blocks)]
    t2 = time.perf_counter()
    for i, j in picks:
        ocons.sample_block(ent, n, p.levels, r, olr.Params(), 0, i, j)
    t_blk = (time.perf_counter() - t2) / len(picks)
    slab = rng.standard_normal((1, side, m, r)) + 1j * rng.standard_normal((1, side, m, r))
    t3 = time.perf_counter()
    ocons.recurse(slab, n, p.levels, r)
    t_slab = time.perf_counter() - t3
    cpu_s = m * m * t_blk + 2 * m * t_slab
    fl = construction_flops(p, r)
    _, dmma, _ = _peaks()
    dfma = LIVE_PEAKS.get("dfma_tflops", 36.43)
    return {"workload": f"{name} factorize {kern.upper()} N={n} r={r} leaf={leaf} (L={p.levels}), sampling mode, "
                        "seed 0, full construction on the GPU",
            "factorize_s": t_fac, "eps_a": eps, "eps_a_s": t_eps, "apply_ms_built": ms,
            "roofline": {"algorithmic_fp64_flops_model": fl, "achieved_tflops": fl / t_fac / 1e12,
                         "dfma_peak_tflops": dfma, "frac_of_fp64_peak": fl / t_fac / 1e12 / dfma,
                         "model": "upper bound: sample sets at their caps r(q+1), bases 3r wide "
                                  "(bench.construction_flops); entry evaluation (sincos) not counted"},
            "cpu_reference": {"factorize_s_extrapolated": cpu_s, "per_block_s": t_blk, "slab_recursion_s": t_slab,
                              "kind": "port", "cores": int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count())),
                              "sample": f"{cpu_blocks} middle blocks x {m * m} + 1 slab recursion x {2 * m}"},
            "speedup_vs_cpu_extrapolated": cpu_s / t_fac,
            "note": "at leaf 16 the reference's own construction diverges as well (its cfg1 eps_a is 3.6e2, "
                    "BASELINE.md; tests/golden/eps_cfg1_*): the configs' inaccuracy comes from the recursion's "
                    "truncation at 16-point leaves, not from the GPU path"}


def run_reference(args):
    """--impl reference: the reference algorithm (NumPy oracle port) on host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    kern, n, r, leaf, k0 = CONFIGS[args.config]
    k = args.rhs or k0
    from paper_1502_01379_b200.synthetic import bench_chain
    p = partition_for(kern, n, leaf)
    weak = args.gpus > 1 and args.scaling == "weak" and kern != "radon2d" and args.config != "cfg4a"
    # the GPU arm's config (at N > 1 with weak scaling the whole job is N = n x GPUs)
    n_job = n * args.gpus if weak else n
    cfg = bench_config(args.config, kern, n_job, r, leaf, k, partition_for(kern, n_job, leaf), "c128",
                       args.gpus, None if args.gpus == 1 else f"node-sharded{args.gpus}")
    fh = bench_chain(p, r, seed=FACTOR_SEED)
    g = rhs_input(n, k)
    from oracle import chain as ochain
    oc = oracle_chain(fh)
    for _ in range(min(args.warmup, 1)):
        ochain.apply(oc, g)
    times = []
    budget = 150.0
    t_all = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ochain.apply(oc, g)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > budget:
            break
    t = statistics.median(times)
    val = n * k / t
    cores = int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1))
    sample = f"{len(times)} full applies of {args.config} (N={n}, r={r}, k={k}), median"
    if weak:
        sample += (f"; the GPU arm runs N={n} per GPU ({n_job} in total, weak scaling): this is one "
                   "GPU's share, timed as the bounded sample of that workload (the CPU would process the "
                   "job's shares one after another at this rate)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": len(times), "warmup": min(args.warmup, 1), "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong" if (args.gpus > 1 and not weak) else "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": val, "unit": "samples/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": val, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def measure_sharded(name, dtype, k, weak, world, rank, local, steps, warm, exchange, e2e=True):
    """One sharded workload on all ranks: each rank owns m/N middle nodes
    per side, runs its down half, the middle factor is an exchange (fused peer stores into
    symmetric memory, or pack + NCCL all-to-all + unpack), then its up half. Device-timed
    with CUDA events, max over ranks; the exchange (or the wait for the peers' stores) is
    timed separately. Returns the fields of a JSON line (rank 0) or None."""
    import torch
    import torch.distributed as dist

    import paper_1502_01379_b200 as bf
    from paper_1502_01379_b200.sharded import PUSH_BARRIER_TIMEOUT_MS, ShardedPlan
    from paper_1502_01379_b200.synthetic import synthetic_slices

    kern, n, r, leaf, _ = CONFIGS[name]
    esz = 16 if dtype == "c128" else 8
    if weak:
        n *= world
    p = partition_for(kern, n, leaf)
    # each rank draws only its own factor slices, on its device (cfg4a: 180 GB in total)
    sp = ShardedPlan(p, r, rank, world, synthetic_slices(p, r, rank, world, seed=FACTOR_SEED, device="cuda"),
                     dtype=dtype)
    torch.cuda.empty_cache()
    tdt = torch.complex128 if dtype == "c128" else torch.complex64
    nl = n // world
    if n * k <= (1 << 24):
        g_host = np.ascontiguousarray(rhs_input(n, k)[rank * nl:(rank + 1) * nl])
    else:   # this rank's rows only, seeded per rank
        rng = np.random.default_rng(np.random.SeedSequence(0, spawn_key=(4, 0, rank)))
        g_host = rng.standard_normal((nl, k)) + 1j * rng.standard_normal((nl, k))
    g = torch.from_numpy(g_host).to("cuda").to(tdt)
    stream = torch.cuda.current_stream()
    if exchange == "push" and world > 1:
        # fused path: validate once against pack + NCCL all-to-all, fall back if unavailable or different
        try:
            ref_out = sp.apply(g)
            push_out = sp.apply_push(g)
            torch.cuda.synchronize()
            ok = torch.equal(ref_out, push_out)
            flag = torch.tensor([1 if ok else 0], device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) != 1:
                exchange = "nccl (push validation failed)"
            del ref_out, push_out
        except Exception as exc:  # symmetric memory / IPC not available
            exchange = f"nccl (push unavailable: {type(exc).__name__})"
    elif exchange == "push":
        exchange = "nccl"      # one rank: nothing to push to
    use_push = exchange == "push"
    run = sp.apply_push if use_push else sp.apply
    for _ in range(warm):
        run(g)
    torch.cuda.synchronize()
    dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(steps):
        if use_push:
            buf, hdl, ptrs = sp.push_buffer(g.shape[1])
            hdl.barrier(timeout_ms=PUSH_BARRIER_TIMEOUT_MS)
            sp.down_push(g, False, ptrs)      # the exchange is fused into this launch's stores
            ev[i][0].record(stream)
            hdl.barrier(timeout_ms=PUSH_BARRIER_TIMEOUT_MS)  # only the wait for the peers' stores is separable
            ev[i][1].record(stream)
            recv = (buf.view(torch.complex128) if sp.tdt == torch.complex128 else buf).view(-1, g.shape[1])
            sp.up(sp.unpack(recv, False), False)
        else:
            mid = sp.down(g, False)
            send = sp.pack(mid, False)
            ev[i][0].record(stream)
            recv = sp.exchange(send)
            ev[i][1].record(stream)
            sp.up(sp.unpack(recv, False), False)
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    t = torch.tensor([e0.elapsed_time(e1), sum(a.elapsed_time(b) for a, b in ev)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step, xch_ms = float(t[0]) / steps, float(t[1]) / steps
    e2e_rec = None
    if e2e:
        # end to end: this rank's pinned host rows in, result rows back to pinned host memory
        g_pin = torch.empty((nl, k), dtype=tdt, pin_memory=True)
        g_pin.copy_(torch.from_numpy(g_host).to(tdt))
        o_pin = torch.empty((nl, k), dtype=tdt, pin_memory=True)
        dist.barrier()
        t0 = time.perf_counter()
        e2e_steps = max(3, min(steps, 10))
        for _ in range(e2e_steps):
            o_pin.copy_(run(g_pin.to("cuda", non_blocking=True)))
        torch.cuda.synchronize()
        e2e_t = torch.tensor([(time.perf_counter() - t0) / e2e_steps], device="cuda")
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        e2e_s = float(e2e_t.item())
        e2e_rec = {"value": n * k / e2e_s, "unit": "samples/s", "h2d_bytes_per_step": n * k * esz,
                   "d2h_bytes_per_step": n * k * esz, "ms_per_step": e2e_s * 1e3}
    del sp, g
    torch.cuda.empty_cache()
    if rank != 0:
        return None
    shapes, leaf_shape = bf.level_geometry(p, r)
    fac_elems = 2 * int(np.prod(leaf_shape)) + 2 * sum(int(np.prod(s_)) for _, _, s_ in shapes)
    nnz_m = p.mid_nodes ** 2 * r
    per_gpu_bytes = esz * fac_elems // world + (esz // 2) * nnz_m + 2 * esz * nl * k
    per_gpu_flops = (8 * k * fac_elems + 2 * k * nnz_m) // world
    a2a_bytes = esz * (world - 1) * sp_chunk_rows(p, r, world) * k
    hbm, dmma, _ = _peaks()
    local_ms = ms_step if use_push else ms_step - xch_ms
    roof = {"achieved_gbs_per_gpu": per_gpu_bytes / (local_ms / 1e3) / 1e9, "hbm_peak": hbm,
            "achieved_tflops_per_gpu": per_gpu_flops / (local_ms / 1e3) / 1e12, "dmma_peak": dmma,
            "kernel": "local chain (down + up) per rank" + (" incl. fused peer stores" if use_push else
                                                            ", exchange excluded")}
    if k < 8:
        roof.update(bound="hbm", achieved=roof["achieved_gbs_per_gpu"], peak=hbm, unit="GB/s",
                    frac=roof["achieved_gbs_per_gpu"] / hbm)
    else:
        roof.update(bound="tensor", achieved=roof["achieved_tflops_per_gpu"], peak=dmma, unit="TFLOP/s",
                    frac=roof["achieved_tflops_per_gpu"] / dmma)
    return {"value": n * k / (ms_step / 1e3), "unit": "samples/s", "n_gpus": world, "steps": steps, "warmup": warm,
            "ms_per_step": ms_step, "config": bench_config(name, kern, n, r, leaf, k, p, dtype, world,
                                                           f"node-sharded{world}"),
            "scaling": "weak" if weak else "strong",
            "sharding": f"middle nodes over {world} GPUs, {'weak scaling: the config per GPU' if weak else 'strong scaling'}"
                        f", exchange at M: {exchange}",
            "exchange": exchange, "a2a_ms_per_step": None if use_push else xch_ms,
            "exchange_wait_ms_per_step": xch_ms if use_push else None, "a2a_bytes_per_rank": a2a_bytes,
            "roofline": roof, "e2e": e2e_rec, "clocks": clk,
            "gpu_launches": (2 * (p.levels - p.half) + (2 if use_push else 4)) * steps}


def sp_chunk_rows(p, r, world):
    mp = p.mid_nodes // world
    return mp * mp * r


def single_gpu_ms(name, k, steps, warm):
    """The unsharded one-GPU apply of a config (the strong-scaling N = 1 point), device-timed."""
    import torch

    from paper_1502_01379_b200.synthetic import synthetic_chain
    kern, n, r, leaf, _ = CONFIGS[name]
    p = partition_for(kern, n, leaf)
    plan = synthetic_chain(p, r, seed=FACTOR_SEED, device="cuda").plan("c128")
    g = torch.from_numpy(rhs_input(n, k)).cuda()
    out = torch.empty_like(g)
    ws = torch.empty(plan.workspace_bytes(k), dtype=torch.uint8, device="cuda")
    ms = dev_time(lambda: plan.apply(g, out=out, workspace=ws), steps, warm)
    del plan, g, out, ws
    torch.cuda.empty_cache()
    return ms


def run_sharded(args, world, rank, local):
    """N > 1 (or --sharded): the headline workload sharded over the ranks — weak scaling by
    default (cfg2 per GPU, N = 2^20 x GPUs), so the driver's per-N values compare — plus,
    in `also`, BASELINE configs[4]: cfg4b (2-D n = 1024, 16 RHS) strong over the N GPUs with
    its one-GPU time and scaling efficiency, and cfg4a (N = 2^24, 64 RHS, 180 GB of
    factors: never on one GPU) at N >= 2, each with the exchange time broken out."""
    import torch
    import torch.distributed as dist

    kern, _, _, _, k0 = CONFIGS[args.config]
    k = args.rhs or k0
    weak = args.scaling == "weak" and kern != "radon2d" and args.config != "cfg4a"
    steps, warm = args.steps, max(args.warmup, 3)
    rec = measure_sharded(args.config, args.dtype, k, weak, world, rank, local, steps, warm, args.exchange)
    also = None
    if not args.no_also and args.config == "cfg2":
        also = {}

        def run(key, fn):
            try:
                res = fn()
            except Exception as exc:   # a companion must not cost the headline line
                res = {"error": f"{type(exc).__name__}: {exc}"[:300]}
            if rank == 0:
                also[key] = res

        def cfg4b():
            res = measure_sharded("cfg4b", "c128", 16, False, world, rank, local, max(3, min(steps, 10)), 3,
                                  args.exchange, e2e=False)
            one = torch.tensor([single_gpu_ms("cfg4b", 16, 5, 3) if rank == 0 else 0.0], device="cuda")
            dist.broadcast(one, 0)
            if res is not None:
                res["one_gpu_ms_per_step"] = float(one.item())
                res["scaling_efficiency"] = float(one.item()) / (world * res["ms_per_step"])
            return res

        run("cfg4b_strong", cfg4b)
        free = torch.tensor([torch.cuda.mem_get_info()[0]], device="cuda", dtype=torch.float64)
        dist.all_reduce(free, op=dist.ReduceOp.MIN)
        # cfg4a: 180.5 GB of factors / N per GPU, ~10 vector buffers of 2^24 x 64 / N complex128
        # (input, middle, send, receive, unpacked, output, ...) and up to two full-length
        # workspace vectors; skipped (on every rank alike) rather than risking one rank's OOM
        # while the others wait in a collective
        need = (180.5e9 + 10 * 17.2e9) / world + 2 * 17.2e9
        if world >= 2 and float(free.item()) > 1.1 * need:
            run("cfg4a_strong", lambda: measure_sharded("cfg4a", "c128", 64, False, world, rank, local,
                                                         max(3, min(steps, 5)), 2, args.exchange, e2e=False))
        elif rank == 0:
            also["cfg4a_strong"] = {"skipped": f"needs ~{need / 1e9:.0f} GB per GPU at {world} GPUs "
                                               f"({float(free.item()) / 1e9:.0f} GB free)"}
    if rank == 0:
        out = {"metric": METRIC, **rec, "higher_is_better": True, "vs_baseline": None, "dtype": args.dtype,
               "data": "synthetic", "cpu_baseline": None, "also": also}
        print(json.dumps(out))
    dist.destroy_process_group()


def _ncu_traffic(config, dtype, k):
    """dram__bytes_read.sum + dram__bytes_write.sum per level-kernel launch from the committed
    `ncu --set full` capture of this workload (profiles/r01_level_kernel_traffic.json), else None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02_level_kernel_traffic.json")
    if (config, dtype, k) != ("cfg2", "c128", 1) or not os.path.exists(path):
        return None
    with open(path) as fh:
        return json.load(fh).get("traffic_bytes_per_launch")


def main():
    args = parse()
    if args.impl == "reference":
        os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count() or 1))
        os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_1502_01379_b200 as bf
    from paper_1502_01379_b200 import _lib
    from paper_1502_01379_b200.synthetic import bench_chain

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 or args.sharded:
        os.environ["NCCL_DEBUG"] = "WARN"   # keep stdout to the one JSON line
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local), rank=rank, world_size=world)
        return run_sharded(args, world, rank, local)
    kern, n, r, leaf, k0 = CONFIGS[args.config]
    k = args.rhs or k0
    esz = 16 if args.dtype == "c128" else 8
    p = partition_for(kern, n, leaf)
    # host-drawn factors, byte-identical to the reference arm's (bench_chain), uploaded once
    f = bench_chain(p, r, seed=FACTOR_SEED)
    plan = f.plan(args.dtype)
    lib = _lib.load()
    tdt = torch.complex128 if args.dtype == "c128" else torch.complex64
    g_host = rhs_input(n, k)
    g = torch.from_numpy(g_host).to("cuda").to(tdt)
    out = torch.empty_like(g)
    wsb = plan.workspace_bytes(k)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    steps, warm = args.steps, max(args.warmup, 3)

    def apply_once(timer=None):
        if timer is None:
            _lib.check(lib.bf_apply(plan._h, ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(out.data_ptr()), k, 0,
                                    ctypes.c_void_p(ws.data_ptr()), wsb, sp))
        else:
            _lib.check(lib.bf_apply_timed(plan._h, ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(out.data_ptr()), k,
                                          0, ctypes.c_void_p(ws.data_ptr()), wsb, sp, timer))

    for _ in range(warm):
        apply_once()
    torch.cuda.synchronize()
    live = None
    if world == 1:
        try:
            live = measure_live_peaks()
        except Exception as exc:  # the file values stand in
            live = {"error": f"{type(exc).__name__}: {exc}"[:200]}
        for _ in range(warm):   # back to the apply's steady state after the peak kernels
            apply_once()
        torch.cuda.synchronize()

    nlaunch = 2 + 2 * len(f.g_chain)
    # timed region: K applies through bf_apply (the chain replays as one CUDA graph)
    apply_once()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        apply_once()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / steps
    # per-launch breakdown: the same K steps again with CUDA events around every launch
    # (bf_apply_timed, on the launch stream); the dominant kernel's roofline comes from it
    timer = ctypes.c_void_p()
    _lib.check(lib.bf_timer_create(ctypes.byref(timer), steps, nlaunch))
    torch.cuda.synchronize()
    i0, i1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    i0.record(stream)
    for _ in range(steps):
        apply_once(timer)
    i1.record(stream)
    torch.cuda.synchronize()
    instrumented_ms = i0.elapsed_time(i1) / steps
    launch_ms = (ctypes.c_float * (steps * nlaunch))()
    ns, nl = ctypes.c_uint32(), ctypes.c_uint32()
    _lib.check(lib.bf_timer_read(timer, launch_ms, ctypes.byref(ns), ctypes.byref(nl)))
    lib.bf_timer_destroy(timer)
    per_launch = np.array(launch_ms[:steps * nl.value]).reshape(steps, nl.value).mean(axis=0)
    alg_bytes, alg_flops = algorithmic(f, k, esz)
    node = nl.value == 2      # node kernels: each half of the chain is one launch
    if node:
        nlaunch = 2
        lb = [("down half (node kernel)", alg_bytes // 2), ("up half (node kernel)", alg_bytes // 2)]
        lf_all = [("down half (node kernel)", alg_flops // 2), ("up half (node kernel)", alg_flops // 2)]
    else:
        radix4 = nl.value == len(f.g_chain)         # many-RHS twin: pairs of levels folded (plan_build_radix4)
        folded = radix4 or nl.value == 2 * len(f.g_chain)    # leaf factors folded into the outermost levels
        if folded:
            nlaunch = nl.value
        lb = launch_bytes(f, k, esz, folded)
        lf_all = launch_flops(f, k, folded)
        if radix4:   # one launch per pair of reference levels; the vector between them is never moved
            dim = f.g_chain[0].shape[0]
            lb = [(f"{a[0]} + {b[0]}", a[1] + b[1] - 2 * esz * k * dim) for a, b in zip(lb[0::2], lb[1::2])]
            lf_all = [(f"{a[0]} + {b[0]}", a[1] + b[1]) for a, b in zip(lf_all[0::2], lf_all[1::2])]
    moved_bytes = alg_bytes
    if not node and folded:
        nb_, n0_, r_ = f.u_outer.blocks.shape
        last = f.g_chain[-1].nnz
        moved_bytes = alg_bytes - esz * 2 * nb_ * n0_ * r_ - esz * 2 * last + esz * 2 * (last // r_) * n0_
    dominant = (lambda name: True) if node else (lambda name: name[0] in "GH")
    peaks = {}
    pk_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk_path):
        peaks = json.load(open(pk_path))
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    # dominant kernel: the transfer-level launches (2*(L-h) of the 2+2(L-h) launches)
    tr = [(name, b, t) for (name, b), t in zip(lb, per_launch) if dominant(name)]
    tr_bytes = sum(b for _, b, _ in tr) / len(tr)
    tr_ms = sum(t for _, _, t in tr) / len(tr)
    share = sum(t for _, _, t in tr) / max(per_launch.sum(), 1e-9)
    roof = {"bound": "hbm", "achieved": tr_bytes / (tr_ms / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
            "frac": tr_bytes / (tr_ms / 1e3) / 1e9 / hbm_peak,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"}
    # the levels are read-dominated (factor blocks read once, vectors L2-resident): their own
    # ceiling is the streaming-read bandwidth, measured in this process (bf_measure_peaks)
    _, _, rd = _peaks()
    roof.update(read_peak=rd, frac_of_read_peak=roof["achieved"] / rd,
                read_peak_source=("bf_measure_peaks in this run" if "read_gbs" in LIVE_PEAKS else
                                  "profiles/r01_fp64_peaks.json read_gbs") +
                " (MEASURED_PEAKS.json hbm_gbs is a copy: half reads, half writes)")
    if k >= 8 and args.dtype == "c128":
        # many right-hand sides: the transfer levels are FP64 tensor-core (DMMA) bound
        # (SURVEY.md §8(d)); algorithmic flops (8 per complex multiply-add) per launch
        tr_fl = sum(fl for (name, fl) in lf_all if dominant(name)) / len(tr)
        _, dmma_peak, _ = _peaks()
        roof = {"bound": "tensor", "achieved": tr_fl / (tr_ms / 1e3) / 1e12, "peak": dmma_peak, "unit": "TFLOP/s",
                "frac": tr_fl / (tr_ms / 1e3) / 1e12 / dmma_peak,
                "peak_source": ("bf_measure_peaks in this run" if "dmma_tflops" in LIVE_PEAKS else
                                "profiles/r01_fp64_peaks.json") +
                               " (FP64 tensor pipe, mma.sync m8n8k4; MEASURED_PEAKS.json has no FP64 figure)",
                "note": "complex products run as 3 real DMMAs (Gauss form), so the algorithmic rate can exceed "
                        "the 4-product tensor-pipe rate by up to 4/3"}

    # end to end through the public API with pinned host buffers
    g_pin = torch.empty((n, k), dtype=tdt, pin_memory=True)
    g_pin.copy_(torch.from_numpy(g_host).to(tdt))
    o_pin = torch.empty((n, k), dtype=tdt, pin_memory=True)
    g_np, o_np = g_pin.numpy(), o_pin.numpy()
    for _ in range(max(20, warm)):  # host-side warm-up too (first transfers on a fresh box are slow)
        plan.apply(g_np, out=o_np)
    e2e_steps = max(10, min(steps, 30))
    if world > 1:
        dist.barrier()
    # each public apply is synchronous (H2D + chain + D2H, result back in host memory):
    # per-step wall times, median (host-side jitter of single steps is not the path's cost)
    e2e_times = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        plan.apply(g_np, out=o_np)
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = float(np.median(e2e_times))
    e2e_mean_s = float(np.mean(e2e_times))
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    cpu = None
    rel_err = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the reference algorithm (oracle port) on the identical factors and right-hand sides:
        # the CPU baseline's timing, and the GPU output's relative error against it
        os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count() or 1))
        cpu_k = min(k, 16)
        t_cpu, nrun, want = time_cpu(f, g_host[:, :cpu_k].astype(np.complex128))
        got = out[:, :cpu_k].cpu().numpy().astype(np.complex128)
        rel_err = {"value": rel2(got, want), "columns": cpu_k,
                   "tolerance": 1e-11 if args.dtype == "c128" else 1e-5,
                   "against": "oracle port of ButterflyFactors.apply (CPU, float64) on the identical factors "
                              "and inputs"}
        cpu = {"value": n * cpu_k / t_cpu, "unit": "samples/s", "cores": int(os.environ["OPENBLAS_NUM_THREADS"]),
               "kind": "port",
               "sample": f"oracle port of ButterflyFactors.apply on the identical factors, k={cpu_k}, "
                         f"median of {nrun} applies ({t_cpu:.2f} s each); the path is effectively single-core"}

    # companion workloads (BASELINE configs[1]-[3]), each device-timed with its own parity check
    also = None
    if rank == 0 and world == 1 and args.config == "cfg2" and not args.no_also:
        del ws
        torch.cuda.empty_cache()
        also = {}

        def run(name, fn, *a):
            try:
                also[name] = fn(*a)
            except Exception as exc:   # a companion must not cost the headline line
                also[name] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
            torch.cuda.empty_cache()

        run("cfg0_k1", companion_cfg, "cfg0", "c128", 0, steps, warm)
        run("cfg1_k64", companion_cfg, "cfg1", "c128", 0, steps, warm)
        if args.dtype == "c128" and k == 1:
            run("cfg2_k256", companion_many_rhs, plan, f, n, steps, warm)
            run("cfg2_c64_k1", companion_same_plan_c64, f, n, steps, warm)
        del plan
        torch.cuda.empty_cache()
        run("cfg3_k16", companion_cfg, "cfg3", "c128", 0, steps, warm)
        run("cfg4b_k16", companion_cfg, "cfg4b", "c128", 0, steps, warm)
        run("cfg2_construction", companion_construction, "cfg2")

    if rank == 0:
        total = n * k * world
        rec = {
            "metric": METRIC, "value": total / (ms_step / 1e3), "unit": "samples/s", "n_gpus": world,
            "steps": steps, "warmup": warm, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": bench_config(args.config, kern, n, r, leaf, k, p, args.dtype, world),
            "rel_err": rel_err,
            "roofline": dict(roof, traffic=_ncu_traffic(args.config, args.dtype, k),
                             kernel="node_kernel (one launch per half)" if node else
                             ("wide_kernel (branching-4 twin: pairs of transfer levels)" if (not node and radix4)
                              else "level_kernel (transfer levels G/H)"), kernel_share_of_step=share),
            "chain_roofline": {"algorithmic_bytes": alg_bytes, "algorithmic_flops": alg_flops,
                               "moved_bytes": moved_bytes,
                               "achieved_gbs": moved_bytes / (ms_step / 1e3) / 1e9,
                               "frac": moved_bytes / (ms_step / 1e3) / 1e9 / hbm_peak,
                               "note": "algorithmic_bytes is SURVEY 8(d)'s figure for the reference's factor list; "
                                       "achieved uses moved_bytes, the compulsory bytes of the chain as launched "
                                       "(leaf factors folded into the outermost levels at plan upload: the two leaf "
                                       "factors are never read, the folded blocks are n0 x C)"},
            "per_launch_ms": {name: round(float(t), 5) for (name, _), t in zip(lb, per_launch)},
            "ms_per_step_instrumented": instrumented_ms,
            "e2e": {"value": total / e2e_s, "unit": "samples/s", "h2d_bytes_per_step": n * k * esz,
                    "d2h_bytes_per_step": n * k * esz, "ms_per_step": e2e_s * 1e3,
                    "ms_per_step_mean": e2e_mean_s * 1e3, "steps": e2e_steps,
                    "method": "ButterflyFactors.apply on pinned host arrays (bf_apply_host: tapered-part H2D/chain/D2H "
                              "pipeline), median of per-step wall times"},
            "gpu_launches": nlaunch * steps,
            "clocks": clk,
            "live_peaks": live,
            "cpu_baseline": cpu,
            "also": also,
        }
        print(json.dumps(rec))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
