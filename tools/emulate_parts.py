"""Per-GPU work of a P-GPU sharded apply, measured on ONE GPU (no peers): part 0's plan
(its 1/P of the factors, drawn directly with `synthetic_slices`) runs its down half, the
middle pack, a same-size local copy standing in for the all-to-all, the unpack and its up
half, timed with CUDA events. This is the compute each GPU of a P-GPU job does; the
NVLink exchange is not measured (every gpurun box has one GPU) and is reported as bytes
plus an estimate at an assumed per-direction bandwidth.

Usage: python tools/emulate_parts.py cfg4a|cfg4b|cfg2 --parts 4 8 [--rhs K] [--steps S]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1502_01379_b200 as bf  # noqa: E402
from paper_1502_01379_b200.sharded import ShardedPlan  # noqa: E402
from paper_1502_01379_b200.synthetic import synthetic_slices  # noqa: E402

CFG = {"cfg2": ("fio", 1 << 20, 16, 16, 1), "cfg4a": ("fio", 1 << 24, 16, 16, 64),
       "cfg4b": ("radon2d", 1 << 20, 25, 4, 16)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(CFG))
    ap.add_argument("--parts", type=int, nargs="+", default=[8])
    ap.add_argument("--rhs", type=int, default=0)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--nvlink-gbs", type=float, default=700.0, help="assumed per-direction exchange bandwidth")
    args = ap.parse_args()
    kind, n, r, leaf, k0 = CFG[args.config]
    k = args.rhs or k0
    p = bf.make_quadtree_partition(int(round(n ** 0.5)), leaf) if kind == "radon2d" else bf.make_partition(n, leaf)
    for P in args.parts:
        sp = ShardedPlan(p, r, 0, P, synthetic_slices(p, r, 0, P, device="cuda"))
        torch.cuda.empty_cache()
        g = torch.randn((sp.n_local, k), dtype=torch.complex128, device="cuda")

        def step():
            send = sp.pack(sp.down(g, False), False)
            recv = torch.empty_like(send)
            recv.copy_(send)                      # stands in for the all-to-all
            return sp.up(sp.unpack(recv, False), False)

        for _ in range(2):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        sent = (P - 1) / P * sp.mid_rows * k * 16
        est = sent / (args.nvlink_gbs * 1e9) * 1e3
        print(json.dumps({"config": args.config, "n": p.n, "rank": r, "rhs": k, "parts": P,
                          "per_gpu_compute_ms": ms, "exchange_bytes_per_gpu": sent,
                          "exchange_ms_estimate": est, "assumed_nvlink_gbs": args.nvlink_gbs,
                          "job_samples_per_s_estimate": p.n * k / ((ms + est) / 1e3),
                          "note": "part 0 of P on one GPU; identity copy in place of the all-to-all"}))
        del sp, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
