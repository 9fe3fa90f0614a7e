"""One rank of the BNS_TRANSPORT_IPC test (tests/test_gpu_peer.py): launched by torchrun, every rank on cuda:0, a gloo
group carries the host all-gather of the CUDA IPC handles; writes this rank's per-epoch results to <out>_<rank>.npz."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2203_10983_b200 import bns  # noqa: E402
from paper_2203_10983_b200 import inputs as I  # noqa: E402
from test_gpu_parity import wl  # noqa: E402


def main():
    a = json.loads(sys.argv[1])
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    indptr, indices, part, X, y = wl(**a["wl"])
    dims, layer, prec = a["dims"], a["layer"], a["prec"]
    inner = np.nonzero(part == rank)[0]
    ctx = bns.Context(rank=rank, world=world, dims=dims, layer=layer, precision=prec, indptr=indptr,
                      indices=indices, part_of=part, features=np.ascontiguousarray(X[inner]),
                      labels=np.ascontiguousarray(y[inner]), device=0, transport=bns.BNS_TRANSPORT_IPC,
                      allgather=bns.torch_allgather(world), flags=bns.BNS_RETAIN_GRADS)
    W = [torch.tensor(w, device="cuda") for w in I.weights(dims, layer)]
    G = [torch.zeros_like(w) for w in W]
    res = {}
    for e, (kind, p) in enumerate(a["draws"]):
        if kind == "bns":
            ctx.sample_boundary(p, I.BNS_SEED, e)
        else:
            ctx.sample_edges(int(kind), p, I.BNS_SEED, e)
        loss, acc = ctx.epoch(W, 0.3, G)
        torch.cuda.synchronize()
        res[f"loss{e}"] = np.float64(loss)
        res[f"acc{e}"] = np.float64(acc)
        for l in range(len(dims) - 1):
            res[f"g{e}_{l}"] = G[l].cpu().numpy()
            res[f"w{e}_{l}"] = W[l].cpu().numpy()
        for l in range(1, len(dims)):
            res[f"h{e}_{l}"] = ctx.rows(bns.BNS_Q_H, l, dims[l])
            res[f"dh{e}_{l}"] = ctx.rows(bns.BNS_Q_DH, l, dims[l])
    dist.barrier()   # nobody unmaps a buffer a peer may still read
    ctx.close()
    dist.barrier()
    np.savez(f"{a['out']}_{rank}.npz", **res)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
