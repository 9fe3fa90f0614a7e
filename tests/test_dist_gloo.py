"""Multi-process host logic on CPU (world_size 2, gloo, 127.0.0.1): every rank builds its own plan through the C ABI
(BNS_PLAN_ONLY), and real inter-process messages check what the NCCL path relies on without exchanging indices:

* D_{i->j} (what rank i will send) equals the owner-i segment of rank j's boundary list B_j (R24);
* the recomputed send lists S_{i,j} = {u in D_{i->j} : keep(u, j)} equal the owner-i segment of U_j (Alg.1 l.6-7,
  R27) -- the draw here is the oracle's Philox (test infrastructure), the GPU draw is checked bit-exact elsewhere;
* per-peer row counts agree pairwise (the NCCL send/recv sizes);
* bench.py's max-over-ranks timing reduction;
* f1 peer memory: the owner-row map the fused pull reads through (V_j[B_row[b]] == B[b]) and the host all-gather
  callback that carries the CUDA IPC handles (bns.torch_allgather) called through its C function pointer.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, N, nnz, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import oracle as O
        from paper_2203_10983_b200 import bns
        from paper_2203_10983_b200 import inputs as I
        import bench

        indptr, indices = I.rmat(N, nnz, seed=17)
        part = I.partition(indptr, indices, world, "ldg2")
        n_in = int((part == rank).sum())
        ctx = bns.Context(rank=rank, world=world, dims=[4, 2], layer=0, precision=bns.BNS_FP32, indptr=indptr,
                          indices=indices, part_of=part, features=np.zeros((n_in, 4), np.float32),
                          labels=np.zeros(n_in, np.int32), flags=bns.BNS_PLAN_ONLY)
        B = ctx.i32(bns.BNS_Q_BOUNDARY)
        Boff = ctx.i64(bns.BNS_Q_BOUNDARY_OFF)
        D = ctx.i32(bns.BNS_Q_SENDCAND)
        Doff = ctx.i64(bns.BNS_Q_SENDCAND_OFF)
        mine = {"B": B.tolist(), "Boff": Boff.tolist(), "D": D.tolist(), "Doff": Doff.tolist()}
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        for j in range(world):
            if j == rank:
                continue
            theirs = allp[j]
            seg = theirs["B"][theirs["Boff"][rank]:theirs["Boff"][rank + 1]]
            assert mine["D"][mine["Doff"][j]:mine["Doff"][j + 1]] == seg
        # sampled send lists by recomputation vs the receiver's U_j, exchanged point to point
        T = O.threshold(0.3)
        seed = I.BNS_SEED
        for e in range(3):
            S = {j: [u for u in mine["D"][mine["Doff"][j]:mine["Doff"][j + 1]] if O.draw(u, j, e, seed) < T]
                 for j in range(world) if j != rank}
            U = [u for u in mine["B"] if O.draw(u, rank, e, seed) < T]
            Uoff = [0]
            for j in range(world):
                seg = mine["B"][mine["Boff"][j]:mine["Boff"][j + 1]]
                Uoff.append(Uoff[-1] + sum(1 for u in seg if O.draw(u, rank, e, seed) < T))
            for j in range(world):
                if j == rank:
                    continue
                # send my S_{rank,j} to j, receive S_{j,rank} from j (ordered to avoid deadlock)
                out = torch.tensor(S[j] + [-1], dtype=torch.int64)
                n_out = torch.tensor([len(S[j])], dtype=torch.int64)
                n_in_t = torch.zeros(1, dtype=torch.int64)
                if rank < j:
                    dist.send(n_out, j)
                    dist.recv(n_in_t, j)
                else:
                    dist.recv(n_in_t, j)
                    dist.send(n_out, j)
                got = torch.zeros(int(n_in_t.item()) + 1, dtype=torch.int64)
                if rank < j:
                    dist.send(out, j)
                    dist.recv(got, j)
                else:
                    dist.recv(got, j)
                    dist.send(out, j)
                assert got[:-1].tolist() == U[Uoff[j]:Uoff[j + 1]]
        # f1: owner rows of the boundary nodes, checked against the owners' own V lists
        Brow = ctx.i32(bns.BNS_Q_BOUNDARY_ROW)
        V = ctx.i32(bns.BNS_Q_INNER).tolist()
        allV = [None] * world
        dist.all_gather_object(allV, V)
        for j in range(world):
            for b in range(Boff[j], Boff[j + 1]):
                assert allV[j][Brow[b]] == B[b]
        # f1: the IPC host all-gather through its ctypes function pointer (what libbns calls)
        import ctypes
        fn = bns.torch_allgather(world)
        cfn = ctypes.cast(fn, ctypes.c_void_p).value
        call = bns.ALLGATHER_FN(cfn)
        for nb in (67, 4999, 1 << 20):   # small and large (a dangling temporary only shows on large copies)
            send = ((np.arange(nb) * 7 + rank * 50) % 251).astype(np.uint8)
            recv = np.zeros(nb * world, np.uint8)
            assert call(send.ctypes.data, recv.ctypes.data, nb, None) == 0
            for j in range(world):
                assert np.array_equal(recv[j * nb:(j + 1) * nb], ((np.arange(nb) * 7 + j * 50) % 251).astype(np.uint8))
        # max over ranks
        m = bench.max_over_ranks(float(rank + 1) * 1.5, dist, "cpu")
        assert m == 1.5 * world
        ctx.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except BaseException as ex:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))
        raise


@pytest.mark.parametrize("N,nnz", [(400, 4000), (2000, 30000)])
def test_two_process_plan_and_recompute(N, nnz):
    world = 2
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = free_port()
    procs = [ctxm.Process(target=worker, args=(r, world, port, N, nnz, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r, msg in res:
        assert msg == "ok", msg
