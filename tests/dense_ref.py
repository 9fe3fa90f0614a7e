"""Dense-adjacency brute force in float64 with torch autograd -- the independent pin for the oracle.

It never partitions and never exchanges: it writes the sampled propagation of every inner node v as one dense
row of an N x N matrix M (coefficients c_u/deg_G(v) for SAGE, PAPER.md:100 + :335 under readings R1-R3; or
c_u/sqrt(d~_v d~_u) plus the self loop 1/d~_v for GCN, App. A) and lets autograd produce the
backward.  A mistake in the oracle's partitioning, exchange, reverse exchange, accumulation order or hand-written
backward therefore shows up as a mismatch here.
"""
import numpy as np
import torch


def dense_matrix(indptr, indices, part_of, kept, p, layer, arcs=None):
    """kept[i] = set of boundary gids sampled by partition i.  arcs (edge samplers, f3): dict (v, u) -> column
    scale of every arc in the sampled graph; arcs absent from it are dropped (kept/p are then ignored)."""
    N = len(indptr) - 1
    M = np.zeros((N, N))
    deg = np.diff(indptr)
    for v in range(N):
        i = part_of[v]
        for u in indices[indptr[v]:indptr[v + 1]]:
            if arcs is not None:
                c = arcs.get((v, int(u)))
                if c is None:
                    continue
            elif part_of[u] == i:
                c = 1.0
            elif u in kept[i]:
                c = 1.0 / p
            else:
                continue
            if layer == 0:
                M[v, u] += c / deg[v]
            else:
                M[v, u] += c / np.sqrt((deg[v] + 1.0) * (deg[u] + 1.0))
        if layer == 1:
            M[v, v] += 1.0 / (deg[v] + 1.0)
    return M


def forward_backward(indptr, indices, part_of, kept, p, layer, X, labels, Ws, masks=None, arcs=None, targets=None):
    """masks[l]: optional N x d_l elementwise factors on the input of layer l+1 (dropout, R38)."""
    M = torch.tensor(dense_matrix(indptr, indices, part_of, kept, p, layer, arcs), dtype=torch.float64)
    H = torch.tensor(np.asarray(X, np.float64))
    W = [torch.tensor(np.asarray(w, np.float64), requires_grad=True) for w in Ws]
    y = torch.tensor(np.asarray(labels, np.int64))
    L = len(W)
    Hs, Zs = [H], []
    for l in range(L):
        Xin = Hs[-1] if masks is None else Hs[-1] * torch.tensor(masks[l], dtype=torch.float64)
        Z = M @ Xin
        Zs.append(Z)
        pre = torch.cat([Z, Xin], dim=1) @ W[l] if layer == 0 else Z @ W[l]
        Hn = torch.relu(pre) if l < L - 1 else pre
        Hn.retain_grad()
        Hs.append(Hn)
    train = y >= 0
    ntr = int(train.sum())
    logits = Hs[-1]
    if targets is not None:   # f4: multi-label, torch's BCE-with-logits (mean) and sklearn's F1-micro (independent)
        T = torch.tensor(np.asarray(targets, np.float64))
        loss = (torch.nn.functional.binary_cross_entropy_with_logits(logits[train], T[train], reduction="mean")
                if ntr else logits.sum() * 0.0)
        loss.backward()
        from sklearn.metrics import f1_score
        pred = (logits.detach().numpy()[train.numpy()] > 0).astype(int)
        acc = float(f1_score(np.asarray(targets)[train.numpy()], pred, average="micro", zero_division=0)) if ntr else 0.0
    else:
        if ntr:
            loss = torch.nn.functional.cross_entropy(logits[train], y[train], reduction="sum") / ntr
        else:
            loss = logits.sum() * 0.0
        loss.backward()
        am = logits.detach().numpy().argmax(1)  # numpy argmax: first max = lowest index (R22)
        acc = float(((am == y.numpy()) & train.numpy()).sum()) / ntr if ntr else 0.0
    return dict(loss=float(loss.detach()), acc=acc, H=[h.detach().numpy() for h in Hs], Z=[z.detach().numpy() for z in Zs],
                dH=[None] + [h.grad.numpy() if h.grad is not None else None for h in Hs[1:]],
                dW=[w.grad.numpy() for w in W])


def gat_forward_backward(indptr, indices, part_of, kept, X, labels, Ws):
    """f4 / R45 brute force: dense masked GAT (one head, self loops, LeakyReLU 0.2, softmax over the sampled
    neighbourhood), W^l = [W ; a_l ; a_r] ((d_in + 2) x d_out), torch autograd for the backward."""
    N = len(indptr) - 1
    mask = np.zeros((N, N), bool)
    for v in range(N):
        i = part_of[v]
        mask[v, v] = True
        for u in indices[indptr[v]:indptr[v + 1]]:
            if part_of[u] == i or u in kept[i]:
                mask[v, u] = True
    Mk = torch.tensor(mask)
    H = torch.tensor(np.asarray(X, np.float64))
    W = [torch.tensor(np.asarray(w, np.float64), requires_grad=True) for w in Ws]
    y = torch.tensor(np.asarray(labels, np.int64))
    Hs = [H]
    for l in range(len(W)):
        din = Hs[-1].shape[1]
        Y = Hs[-1] @ W[l][:din]
        el = Y @ W[l][din]
        er = Y @ W[l][din + 1]
        E = torch.nn.functional.leaky_relu(el[:, None] + er[None, :], 0.2)
        E = E.masked_fill(~Mk, float("-inf"))
        A = torch.softmax(E, dim=1)
        pre = A @ Y
        Hn = torch.relu(pre) if l < len(W) - 1 else pre
        Hn.retain_grad()
        Hs.append(Hn)
    train = y >= 0
    ntr = int(train.sum())
    logits = Hs[-1]
    loss = torch.nn.functional.cross_entropy(logits[train], y[train], reduction="sum") / ntr
    loss.backward()
    return dict(loss=float(loss.detach()), H=[h.detach().numpy() for h in Hs],
                dH=[None] + [h.grad.numpy() if h.grad is not None else None for h in Hs[1:]],
                dW=[w.grad.numpy() for w in W])
