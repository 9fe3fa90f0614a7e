"""Single-GPU timing emulation of one rank of an m-partition BNS-GCN job (BNS_TRANSPORT_NULL_EMULATE).

The rank runs exactly its own kernels with its own sampled sizes; the exchanges and the all-reduce are no-ops
(their cost is estimated separately from the bytes each would move at the measured 770 GB/s NVLink peer
bandwidth, B200_PROFILING.md).  Output: one JSON line per (p, rank).  This is NOT an 8-GPU measurement; it
exposes per-rank kernel behaviour at the paper's scale (small partitions, launch/latency sensitivity).

    python scripts/emulate_rank.py --m 8 --p 0.1 0.01 --ranks all
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="reddit")
    ap.add_argument("--m", type=int, default=8)
    ap.add_argument("--p", type=float, nargs="+", default=[0.1])
    ap.add_argument("--ranks", default="0")
    ap.add_argument("--prec", default="bf16")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--partition", default="ldg2")
    ap.add_argument("--model", default="sage", choices=["sage", "gat"], help="gat: 2-layer GAT (Table tab:gat)")
    ap.add_argument("--cache-x0", action="store_true", help="BNS_CACHE_INPUT_HALO (f1, R43): no layer-1 exchange")
    ap.add_argument("--no-timing", action="store_true", help="no per-phase CUDA events (device total only)")
    ap.add_argument("--no-prefetch", action="store_true", help="no BNS_PREFETCH_DRAW (R48): draw + host wait per step")
    ap.add_argument("--ceiling", action="store_true",
                    help="also run build/gather_ceiling on this rank's induced forward column stream (one draw)")
    ap.add_argument("--samplers", nargs="+", default=["bns"], choices=["bns", "bes", "dropedge"],
                    help="f3 Table tab:bes analogue: edge samplers at matched dropped-edge counts (P:681)")
    args = ap.parse_args()
    import torch
    from paper_2203_10983_b200 import bns
    from paper_2203_10983_b200 import inputs as I
    sh = I.SHAPES[args.config]
    if args.model == "gat":
        import dataclasses
        sh = dataclasses.replace(sh, layer=I.LAYER_GAT, L=2)
    indptr, indices = I.rmat(sh.N, sh.nnz)
    part = I.partition(indptr, indices, args.m, args.partition)
    y_all = I.labels(sh.N, sh.C, sh.train_frac)
    ranks = list(range(args.m)) if args.ranks == "all" else [int(r) for r in args.ranks.split(",")]
    prec = bns.BNS_BF16 if args.prec == "bf16" else bns.BNS_FP32
    s = 2 if prec == bns.BNS_BF16 else 4
    dp = [((d + 7) // 8) * 8 for d in sh.dims]
    src = np.repeat(np.arange(sh.N, dtype=np.int32), np.diff(indptr))
    cross_frac = float(np.count_nonzero(part[src] != part[indices])) / max(1, len(indices))
    del src
    SAMP = {"bns": bns.BNS_SAMPLER_BNS, "bes": bns.BNS_SAMPLER_BES, "dropedge": bns.BNS_SAMPLER_DROPEDGE}
    for r in ranks:
        inner = np.nonzero(part == r)[0].astype(np.int32)
        ctx = bns.Context(rank=r, world=args.m, dims=sh.dims, layer=sh.layer, precision=prec, indptr=indptr,
                          indices=indices, part_of=part, features=I.features(inner, sh.d0),
                          labels=np.ascontiguousarray(y_all[inner]), transport=bns.BNS_TRANSPORT_NULL_EMULATE,
                          flags=(0 if args.no_timing else bns.BNS_TIMING) | (bns.BNS_CACHE_INPUT_HALO if args.cache_x0 else 0) |
                          (0 if args.no_prefetch else bns.BNS_PREFETCH_DRAW))
        W = [torch.tensor(w, device="cuda") for w in I.weights(sh.dims, sh.layer)]
        G = [torch.zeros_like(w) for w in W]
        stream = torch.cuda.ExternalStream(ctx.stream())
        for p, sname in [(p, sn) for p in args.p for sn in args.samplers]:
            smp = SAMP[sname]
            q = p if smp != bns.BNS_SAMPLER_DROPEDGE else 1.0 - (1.0 - p) * cross_frac

            def one(e):   # one training step (bns_step for BNS: draw + epoch in one C call, as bench.py)
                if smp == bns.BNS_SAMPLER_BNS:
                    ctx.step(p, I.BNS_SEED, e, W, 0.0, G)
                else:
                    ctx.sample_edges(smp, q, I.BNS_SEED, e)
                    ctx.epoch(W, 0.0, G)

            for e in range(args.warmup):
                one(e)
            torch.cuda.synchronize()
            if not args.no_timing:
                ctx.set_timing(False)   # device time without per-phase events (they drain the pipeline)
            k0 = ctx.kernel_count()
            ms = []
            wall0 = time.perf_counter()
            for k in range(args.steps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                one(100 + k)
                b.record(stream)
                b.synchronize()
                ms.append(a.elapsed_time(b))
            wall = (time.perf_counter() - wall0) / args.steps * 1e3
            kern = (ctx.kernel_count() - k0) / args.steps
            if not args.no_timing:   # phase split from a second pass of the same steps with the events on
                ctx.set_timing(True)
            t0 = ctx.times()
            for k in range(args.steps):
                one(200 + k)
            torch.cuda.synchronize()
            t1 = ctx.times()
            cnt = ctx.counts()
            ph = {k: round((t1[k] - t0[k]) / args.steps, 4) for k in t1 if t1[k] - t0[k] > 0}
            # bytes this rank moves per epoch: forward halo rows (recv) and sent rows, backward the reverse
            fwd = sum((cnt["n_halo"] + cnt["n_sent"]) * dp[l] * s for l in range(1 if args.cache_x0 else 0, sh.L)) / 2
            bwd = sum((cnt["n_halo"] + cnt["n_sent"]) * dp[l] * s for l in range(1, sh.L)) / 2
            wbytes = sum(w.numel() * 4 for w in W)
            comm_ms = (fwd + bwd) / 770e9 * 1e3 + 2 * wbytes / 725e9 * 1e3
            # a4 pack reads + writes |S| rows per layer, a12 scatter reads 2 and writes 1 row per returned row
            pack_b = sum(2 * cnt["n_sent"] * dp[l] * s for l in range(1 if args.cache_x0 else 0, sh.L))
            scat_b = sum(3 * cnt["n_sent"] * dp[l] * s for l in range(1, sh.L))
            gbs = lambda b, ph: round(b / (ph * 1e-3) / 1e9, 1) if ph and ph > 0 else None
            rec = {"config": sh.name, "model": args.model, "m": args.m, "rank": r, "p": p, "sampler": sname, "q": q, "prec": args.prec,
                   "pack_gbs": gbs(pack_b, ph.get("pack")), "scatter_gbs": gbs(scat_b, ph.get("scatter")),
                   "cache_x0": bool(args.cache_x0),
                   "device_ms_per_epoch": float(np.median(ms)), "wall_ms_per_epoch": wall,
                   "est_nvlink_ms": comm_ms, "kernels_per_epoch": kern,
                   "n_in": cnt["n_in"], "n_bd": cnt["n_bd"], "n_halo": cnt["n_halo"], "n_sent": cnt["n_sent"],
                   "nnz_kept": cnt["nnz_kept"], "phases_ms": ph,
                   "note": "single-GPU emulation: exchanges/all-reduce are no-ops; NOT an m-GPU measurement"}
            print(json.dumps(rec), flush=True)
            if args.ceiling and smp == bns.BNS_SAMPLER_BNS:
                # the gather ceiling of exactly this rank's forward column stream (CSR order, no row boundaries)
                import subprocess
                import tempfile
                ctx.sample_boundary(p, I.BNS_SEED, 0)
                ptr, cols = ctx.induced(cnt["n_in"])
                exe = os.path.join(ROOT, "build", "gather_ceiling")
                w = dp[1] * s
                with tempfile.TemporaryDirectory() as d:
                    f = os.path.join(d, "col.bin")
                    np.ascontiguousarray(cols, np.int32).tofile(f)
                    for rb, stride, tag in [(w, w, f"{sh.name} m={args.m} rank {r} p={p} induced CSR order, {w} B rows"),
                                            (w, 2 * w, f"{sh.name} m={args.m} rank {r} p={p} induced CSR order, {w} B rows at {2 * w} B stride")]:
                        subprocess.run([exe, "20", f, str(rb), str(stride), tag], check=True)
        ctx.close()


if __name__ == "__main__":
    main()
