"""World-size-2 gloo test (CPU) of the row-sharded Sinkhorn protocol.

Each rank holds a contiguous slice of the source rows (distributed.shard_rows)
and the whole target side.  Per iteration it exchanges exactly what the
CUDA path all-gathers (csrc/sinkhorn.cu run_sharded): one (shift, sum) pair
per column plus the previous f-update's scalar partials; every rank resolves
the translation scalars and folds the column pairs in rank order.  The
reduction arithmetic is the fp64 oracle's; the result must equal the
unsharded oracle H-Sinkhorn."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2201_00730_b200.distributed import row_offset, shard_problems, shard_rows


def _lse_pairs(vals, w, axis):
    """Per-column (max, sum) of w * exp(vals - max) along `axis` (natural domain)."""
    masked = np.where(w > 0, vals, -np.inf)
    m = masked.max(axis=axis)
    s = np.sum(np.where(w > 0, w * np.exp(masked - np.expand_dims(m, axis)), 0.0), axis=axis)
    return m, s


def _merge(ms, ss):
    M = np.max(np.where(ss > 0, ms, -np.inf), axis=0)
    acc = np.sum(np.where(ss > 0, ss * np.exp(ms - M), 0.0), axis=0)
    return M, acc


def _sharded_h_sinkhorn(rank, world, x, y, a, b, eps, rho, iters, chunks=1):
    n = len(x)
    rows = shard_rows(n, world)
    off = row_offset(n, world, rank)
    xl, al = x[off:off + rows[rank]], a[off:off + rows[rank]]
    C = (xl[:, None] - y[None, :]) ** 2  # local rows x all columns
    r1 = r2 = rho
    kA = (eps / (eps + r1)) * (r2 / (r1 + r2))
    kB = (eps / (eps + r2)) * (r1 / (r1 + r2))
    facA, facB = kA / (1 - kA), kB / (1 - kB)
    aA, aB = r1 / (r1 + eps), r2 / (r2 + eps)
    cA, cB = (eps / (eps + r1)) * (r1 / (r1 + r2)), (eps / (eps + r2)) * (r2 / (r1 + r2))
    hat_a = np.zeros(len(xl))

    def scal(hat, dl):
        m, s = _lse_pairs(-hat / r1, al, 0)
        return np.array([m, s, dl.max() if dl is not None else -np.inf,
                         dl.min() if dl is not None else np.inf])

    def gather(arr):
        t = torch.as_tensor(arr)
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return np.stack([o.numpy() for o in out])

    my_scal = scal(hat_a, None)
    tau_a = 0.0
    hat_g = tau_b = shat_b = None
    deltas = []
    for t in range(iters):
        if chunks == 1:
            m, s = _lse_pairs((hat_a[:, None] - C) / eps, al[:, None], 0)
            allp = gather(np.concatenate([my_scal, m, s]))
            sc, pm, ps = allp[:, :4], allp[:, 4:4 + len(y)], allp[:, 4 + len(y):]
        else:
            # column chunks: chunk c's gather is in flight (async) while chunk
            # c+1 is reduced, as run_sharded overlaps them on a second stream;
            # the scalars travel with chunk 0
            pend = []
            for c in range(chunks):
                c0, c1 = len(y) * c // chunks, len(y) * (c + 1) // chunks
                m, s = _lse_pairs((hat_a[:, None] - C[:, c0:c1]) / eps, al[:, None], 0)
                pay = np.concatenate([my_scal, m, s]) if c == 0 else np.concatenate([m, s])
                tt = torch.as_tensor(pay)
                out = [torch.empty_like(tt) for _ in range(world)]
                pend.append((c0, c1, out, dist.all_gather(out, tt, async_op=True)))
            pm = np.empty((world, len(y)))
            ps = np.empty((world, len(y)))
            for c, (c0, c1, out, work) in enumerate(pend):
                work.wait()
                arr = np.stack([o.numpy() for o in out])
                if c == 0:
                    sc, arr = arr[:, :4], arr[:, 4:]
                w = c1 - c0
                pm[:, c0:c1], ps[:, c0:c1] = arr[:, :w], arr[:, w:]
        qm, qs = _merge(sc[:, 0:1], sc[:, 1:2])
        shat_a = -r1 * (qm[0] + np.log(qs[0]))
        new_tau_a = 0.0 if t == 0 else facA * shat_a
        if t > 0:
            deltas.append(max(sc[:, 2].max() + new_tau_a, -(sc[:, 3].min() + new_tau_a)))
        tau_a = new_tau_a
        M, acc = _merge(pm, ps)
        lse = M + np.log(acc) + tau_a / eps
        hat_g = aB * (-eps * lse) - cB * (shat_a + tau_a)
        shat_b = O.softmin(b, r2, hat_g)
        tau_b = facB * shat_b
        lse_f = O.logdotexp(((hat_g + tau_b)[None, :] - C) / eps, b, axis=1)
        hat_new = aA * (-eps * lse_f) - cA * (shat_b + tau_b)
        my_scal = scal(hat_new, hat_new - (hat_a + tau_a))
        hat_a = hat_new
    sc = gather(my_scal)
    qm, qs = _merge(sc[:, 0:1], sc[:, 1:2])
    tau_a = facA * (-r1 * (qm[0] + np.log(qs[0])))
    deltas.append(max(sc[:, 2].max() + tau_a, -(sc[:, 3].min() + tau_a)))
    return hat_a + tau_a, hat_g + tau_b, np.array(deltas)


def _worker(rank, world, port, q, chunks=1):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(4)
        n, m = 37, 29
        x = np.sort(rng.uniform(0, 1, n))
        y = np.sort(rng.uniform(0, 1, m))
        a = rng.uniform(0.1, 1.0, n)
        b = rng.uniform(0.1, 1.0, m) * 1.3
        f_loc, g, dl = _sharded_h_sinkhorn(rank, world, x, y, a, b, 0.05, 1.0, 30, chunks)
        parts = [None] * world
        dist.all_gather_object(parts, f_loc)
        if rank == 0:
            f = np.concatenate(parts)
            cost = O.PointCost(x, y, power1d=True)
            fo, go, do = O.sinkhorn_fixed(cost, a, b, 0.05, 1.0, 1.0, "h", 30)
            q.put((float(np.abs(f - fo).max()), float(np.abs(g - go).max()),
                   float(np.abs(dl - do).max())))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_partitions():
    assert shard_rows(10, 3) == [4, 3, 3]
    assert sum(shard_rows(65536, 8)) == 65536
    assert row_offset(10, 3, 2) == 7
    assert shard_problems(64, 8, 3) == (24, 32)
    assert shard_problems(4096, 3, 2) == (2731, 4096)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("chunks", [1, 3])
def test_sharded_protocol_gloo_world2(chunks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, chunks)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
    assert all(p.exitcode == 0 for p in procs)
    ef, eg, ed = q.get(timeout=5)
    assert ef < 1e-12 and eg < 1e-12 and ed < 1e-12, (ef, eg, ed)
