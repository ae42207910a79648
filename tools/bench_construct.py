"""Construction timing on the GPU (factorize, sampling mode) with a CPU oracle
comparison on a sample of blocks. Usage:
  python tools/bench_construct.py cfg0|cfg1|cfg2 [--full] [--cpu-blocks N]
cfg2 (65,536 middle blocks) is timed on one block-row plus its slab recursion
and extrapolated (x m block-rows, x 2 slab recursions per row) unless --full.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1502_01379_b200 as bf  # noqa: E402
from paper_1502_01379_b200 import construct as bc  # noqa: E402

CFG = {"cfg0": ("fio", 1 << 10, 12, 8), "cfg1": ("dftp", 1 << 16, 8, 16), "cfg2": ("fio", 1 << 20, 16, 16),
       "comp1024": ("fio", 1 << 10, 12, 0.25), "hk1024": ("hankel", 1 << 10, 6, 0.25),
       "hk4096": ("hankel", 1 << 12, 8, 1)}


def kernel(kind, n):
    return {"fio": bf.FioKernel, "dftp": bf.DftPlusKernel, "hankel": bf.HankelKernel}[kind](n)


def sync_time(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t0, out


def bench_matvec(args):
    """matvec mode on the composition operator K F K (the paper's experiment,
    reference test_acceptance.py:75-96): inner chain K by the GPU sampling
    construction (untimed), then factorize(ComposedOperator(K), mode="matvec")
    timed on the GPU and through the oracle port (== reference, bitwise) on the CPU."""
    from oracle import chain as ochain
    from oracle import construct as ocons
    from oracle import operators as oops
    from paper_1502_01379_b200.synthetic import to_host
    kind, n, r, leaf = CFG[args.config]
    p = bf.make_partition(n, leaf)
    inner = bf.factorize(kernel(kind, n), p, r, seed=7)
    comp = bf.ComposedOperator(inner)
    bf.factorize(comp, p, r, seed=0, mode="matvec")          # warm-up
    t, f = sync_time(lambda: bf.factorize(comp, p, r, seed=0, mode="matvec"))
    eps = bf.estimate_eps_a(f, bf.OperatorReference(comp), 256, np.random.SeedSequence(0, spawn_key=(4, 0)))
    h = to_host(inner)
    chain = ochain.Chain(n, p.levels, r, h.u_outer.blocks, [(x.level, x.blocks) for x in h.g_chain],
                         h.middle.weights, [(x.level, x.blocks) for x in h.h_chain], h.v_outer.blocks)
    t0 = time.perf_counter()
    c = ocons.factorize(oops.Composed(chain), n, p.levels, r, seed=0, mode="matvec")
    t_cpu = time.perf_counter() - t0
    rng = np.random.default_rng(3)
    g = rng.standard_normal((n, 2)) + 1j * rng.standard_normal((n, 2))
    want = ochain.apply(c, g)
    got = f.apply(g)
    res = {"config": args.config, "mode": "matvec", "operator": "ComposedOperator(K F K)", "n": n, "r": r,
           "levels": p.levels, "gpu_factorize_s": t, "cpu_factorize_s": t_cpu,
           "cpu_method": f"oracle port (== reference bitwise), cores={os.cpu_count()}",
           "speedup": t_cpu / t, "eps_a": eps,
           "rel_vs_oracle_chain": float(np.linalg.norm(got - want) / np.linalg.norm(want))}
    print(json.dumps(res))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(CFG))
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--cpu-blocks", type=int, default=4)
    ap.add_argument("--mode", choices=["sampling", "matvec"], default="sampling")
    ap.add_argument("--rows", type=int, default=0, help="cfg2: block-rows per middle launch (default: factorize's)")
    args = ap.parse_args()
    if args.mode == "matvec":
        return bench_matvec(args)
    kind, n, r, leaf = CFG[args.config]
    p = bf.make_partition(n, leaf)
    m, side = p.mid_nodes, p.mid_side
    ker = kernel(kind, n)
    res = {"config": args.config, "n": n, "r": r, "levels": p.levels, "m": m, "side": side}
    # warm-up (module load, first launches)
    bc.MiddleSampler(ker, p, r).blocks([(0, 0)])
    torch.cuda.synchronize()
    if args.full or args.config != "cfg2":
        t, f = sync_time(lambda: bf.factorize(ker, p, r, seed=0))
        res["gpu_factorize_s"] = t
        res["method"] = "full factorize (sampling mode)"
    else:
        ms = bc.MiddleSampler(ker, p, r, seed=0)
        t_draws, _ = sync_time(ms.prepare_draws)          # all 65,536 blocks' tables, process pool
        rows = args.rows or ms.batch_rows()
        ij = [(i, j) for i in range(rows) for j in range(m)]
        ms.blocks(ij)                                       # warm: workspace allocation, first launches
        t_mid, (u, v, w) = sync_time(lambda: ms.blocks(ij))
        t_mid /= rows
        u = u[:m]
        res["gpu_rows_per_launch"] = rows
        kb = bc.recursion_batch(m, side, r)               # slabs per recursion launch (factorize's batching)
        slab = u.permute(1, 0, 2).reshape(1, side, m, r).expand(kb, side, m, r).contiguous()
        bc.recurse(slab, p, r)
        t_rec, _ = sync_time(lambda: bc.recurse(slab, p, r))
        res["gpu_draw_tables_s"] = t_draws
        res["gpu_block_row_s"] = t_mid
        res["gpu_slab_batch"] = kb
        res["gpu_slab_batch_recursion_s"] = t_rec
        res["gpu_factorize_s"] = t_draws + m * t_mid + 2 * m / kb * t_rec
        res["method"] = (f"host draw tables (all blocks) + 1 block-row ({m} blocks) x{m} rows + "
                         f"1 recursion of {kb} slabs x{2 * m // kb} batches (warm timings)")
    # CPU: the reference algorithm (oracle port) on a sample of middle blocks + one slab recursion
    from oracle import construct as ocons
    from oracle import entries as oent
    from oracle import lowrank as olr
    ent = oent.EntryOracle(kind, n)
    if kind == "hankel":
        # the reference's row cache makes per-block samples unrepresentative: time it whole
        t0 = time.perf_counter()
        ocons.factorize(ent, n, p.levels, r, seed=0)
        res["cpu_factorize_s"] = time.perf_counter() - t0
        res["cpu_method"] = f"oracle port (== reference bitwise), full factorize; cores={os.cpu_count()}"
        res["speedup"] = res["cpu_factorize_s"] / res["gpu_factorize_s"]
        print(json.dumps(res))
        return
    rng = np.random.default_rng(0)
    picks = [(int(rng.integers(m)), int(rng.integers(m))) for _ in range(args.cpu_blocks)]
    t0 = time.perf_counter()
    for i, j in picks:
        ocons.sample_block(ent, n, p.levels, r, olr.Params(), 0, i, j)
    t_blk = (time.perf_counter() - t0) / len(picks)
    slab = np.asarray(rng.standard_normal((1, side, m, r)) + 1j * rng.standard_normal((1, side, m, r)))
    t0 = time.perf_counter()
    ocons.recurse(slab, n, p.levels, r)
    t_slab = time.perf_counter() - t0
    res["cpu_per_block_s"] = t_blk
    res["cpu_slab_recursion_s"] = t_slab
    res["cpu_factorize_s_extrapolated"] = m * m * t_blk + 2 * m * t_slab
    res["cpu_method"] = (f"oracle port (reference algorithm), {len(picks)} sampled middle blocks x {m * m} + "
                         f"1 slab recursion x {2 * m}; cores={os.environ.get('OPENBLAS_NUM_THREADS', os.cpu_count())}")
    res["speedup"] = res["cpu_factorize_s_extrapolated"] / res["gpu_factorize_s"]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
