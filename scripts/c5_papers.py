"""C5 (BASELINE.json configs[4]): ogbn-papers100M-shaped R-MAT (111,059,956 nodes, 1.6 B arcs, 128 features,
172 classes), GraphSAGE 3 x 128, m = 8 partitions, p = 0.01 (PAPER.md:549-563 Table tab:papers100m; the model of
PAPER.md:419) -- one rank of the 8-GPU job emulated on ONE B200 (the per-rank data fits a B200; 8 ranks on one
GPU do not).  SURVEY §8(c) "Large-config parity" pins for C5, checked here against the oracle:

* keep masks, U_i and S_{i,j} of the emulated rank bit-exact against the oracle's plan + sample (two epochs);
* 1,000 spot rows of H^(1) of that rank recomputed in float64 from raw neighbours (R1: full-graph degree, kept
  boundary columns x 1/p, CONCAT(z, x) W), restricted to rows whose sampled neighbourhood holds no halo row (the
  emulation's exchanges are no-ops, so halo rows carry no data) -- plus the largest-degree such rows;
* epoch time of the rank (device, CUDA events, bns_step = draw + epoch) with the exchanges as no-ops, and the bytes
  the exchanges would move (their NVLink time estimated separately).

Loss parity is unpinned at C5 (a float64 oracle epoch needs ~10^2 GB per tensor).

    python scripts/c5_papers.py [--ranks 0] [--partition random] [--steps 10] > c5.jsonl
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(ranks=(0,), partition="random", steps=10, warmup=3, spot=1000, log=print):
    import torch

    from oracle import oracle as O
    from paper_2203_10983_b200 import bns
    from paper_2203_10983_b200 import inputs as I
    sh = I.SHAPES["papers"]
    m, p = sh.m, sh.p
    t0 = time.time()
    indptr, indices = I.rmat(sh.N, sh.nnz)
    t_gen = time.time() - t0
    part = I.partition(indptr, indices, m, partition)
    y_all = I.labels(sh.N, sh.C, sh.train_frac)
    t0 = time.time()
    orc = O.Oracle(indptr, indices, part, m, [1, 1], 0, np.zeros((sh.N, 1), np.float32), np.zeros(sh.N, np.int32))
    t_orc = time.time() - t0
    deg = np.diff(indptr)
    dims = sh.dims
    Ws = I.weights(dims, sh.layer)
    out = []
    for r in ranks:
        inner = np.nonzero(part == r)[0].astype(np.int32)
        X = I.features(inner, sh.d0)
        t0 = time.time()
        ctx = bns.Context(rank=r, world=m, dims=dims, layer=sh.layer, precision=bns.BNS_BF16, indptr=indptr,
                          indices=indices, part_of=part, features=X, labels=np.ascontiguousarray(y_all[inner]),
                          transport=bns.BNS_TRANSPORT_NULL_EMULATE, max_p=2 * p, flags=bns.BNS_TIMING | bns.BNS_PREFETCH_DRAW)
        t_setup = time.time() - t0
        try:
            # ---- masks and lists bit-exact (two draws)
            for e in (0, 1):
                ctx.sample_boundary(p, I.BNS_SEED, e)
                orc.sample(p, I.BNS_SEED, e)
                assert np.array_equal(ctx.mask(), orc.list(O.KEEP, r).astype(np.uint8)), ("mask", r, e)
                U = ctx.i32(bns.BNS_Q_HALO)
                assert np.array_equal(U, orc.list(O.U_LIST, r)), ("U", r, e)
                S, So = ctx.i32(bns.BNS_Q_SEND), ctx.i64(bns.BNS_Q_SEND_OFF)
                for j in range(m):
                    assert np.array_equal(S[So[j]:So[j + 1]], orc.list(O.S_LIST, r, j)), ("S", r, e, j)
            # ---- one epoch on the last draw, then spot rows of H^1
            W = [torch.tensor(w, device="cuda") for w in Ws]
            G = [torch.zeros_like(w) for w in W]
            loss, acc = ctx.epoch(W, 0.0, G)
            Us = np.sort(U)
            rng = np.random.default_rng(17)
            halo_free = []
            cand = rng.permutation(len(inner))
            by_deg = np.argsort(-deg[inner])
            for k in np.concatenate([by_deg[:2000], cand]):
                v = int(inner[k])
                nb = indices[indptr[v]:indptr[v + 1]]
                bd = nb[part[nb] != r]
                pos_u = np.searchsorted(Us, bd)
                if not np.any((pos_u < len(Us)) & (Us[np.minimum(pos_u, len(Us) - 1)] == bd)):
                    halo_free.append(int(k))
                if len(halo_free) >= spot:
                    break
            rows = np.array(sorted(set(halo_free)), np.int64)
            H1 = ctx.rows(bns.BNS_Q_H, 1, dims[1])
            W0 = torch.tensor(Ws[0]).bfloat16().double().numpy()     # the bf16 GEMM operand (R19)
            z = np.zeros((len(rows), sh.d0))
            for i, k in enumerate(rows):
                v = int(inner[k])
                nb = indices[indptr[v]:indptr[v + 1]]
                nb = nb[part[nb] == r]
                if deg[v]:   # inner neighbours only (no kept halo column by selection); dropped ones count in deg (R1)
                    z[i] = X[np.searchsorted(inner, nb)].astype(np.float64).sum(0) / deg[v]
            pre = np.concatenate([z, X[rows].astype(np.float64)], 1) @ W0
            h = np.maximum(pre, 0)
            err = float(np.abs(H1[rows] - h).max() / max(np.abs(h).max(), 1e-30))
            assert err < 2e-2, ("spot rows H1", r, err)
            # ---- rank epoch time (exchanges no-ops)
            stream = torch.cuda.ExternalStream(ctx.stream())
            for e in range(warmup):
                ctx.step(p, I.BNS_SEED, 10 + e, W, 0.0, G)
            torch.cuda.synchronize()
            ctx.set_timing(False)   # device time without per-phase events; the phase split from a second pass
            ms = []
            k0 = ctx.kernel_count()
            for k in range(steps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                ctx.step(p, I.BNS_SEED, 100 + k, W, 0.0, G)
                b.record(stream)
                b.synchronize()
                ms.append(a.elapsed_time(b))
            kern = (ctx.kernel_count() - k0) / steps
            ctx.set_timing(True)
            t0p = ctx.times()
            for k in range(steps):
                ctx.step(p, I.BNS_SEED, 200 + k, W, 0.0, G)
            torch.cuda.synchronize()
            t1p = ctx.times()
            phases = {k: round((t1p[k] - t0p[k]) / steps, 3) for k in t1p if t1p[k] - t0p[k] > 0}
            cnt = ctx.counts()
            dp = [((d + 7) // 8) * 8 for d in dims]
            xbytes = sum((cnt["n_halo"] + cnt["n_sent"]) * dp[l] * 2 for l in range(sh.L)) + \
                sum((cnt["n_halo"] + cnt["n_sent"]) * dp[l] * 2 for l in range(1, sh.L))
            rec = {"config": "papers100M-shaped R-MAT", "N": sh.N, "nnz": int(indptr[-1]), "m": m, "rank": r, "p": p,
                   "partition": partition, "prec": "bf16", "model": f"GraphSAGE {sh.L} x {sh.hidden}",
                   "lists_bitexact_epochs": [0, 1], "spot_rows": int(len(rows)), "spot_max_degree": int(deg[inner[rows]].max()),
                   "spot_relerr_H1": err, "loss": loss, "device_ms_per_epoch": float(np.median(ms)),
                   "projected_epochs_per_s_if_slowest": 1000.0 / float(np.median(ms)),
                   "kernels_per_epoch": kern, "phases_ms": phases,
                   "n_in": cnt["n_in"], "n_bd": cnt["n_bd"], "n_halo": cnt["n_halo"], "n_sent": cnt["n_sent"],
                   "nnz_rank": cnt["nnz"], "nnz_kept": cnt["nnz_kept"], "exchange_bytes_per_epoch": int(xbytes),
                   "est_nvlink_ms": xbytes / 770e9 * 1e3, "memory_bytes": ctx.memory()[0],
                   "setup_s": t_setup, "graph_gen_s": t_gen, "oracle_plan_s": t_orc,
                   "note": "one rank of the m = 8 job on one B200; exchanges / all-reduce are no-ops (timing "
                           "emulation); lists bit-exact vs the oracle; H1 spot rows vs float64 from raw neighbours"}
            log(json.dumps(rec))
            out.append(rec)
        finally:
            ctx.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", default="0")
    ap.add_argument("--partition", default="random", choices=["random", "ldg2"])
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    run([int(r) for r in args.ranks.split(",")], args.partition, args.steps, log=lambda s: print(s, flush=True))


if __name__ == "__main__":
    main()
