"""The N > 1 path on CPU with gloo, world size 2 (no GPU needed).

(1) bench.py's multi-rank plumbing: process-group setup, barrier, max-over-ranks
    timing and the weak-scaling aggregate.
(2) The channel decomposition's arithmetic contract across processes: each rank
    owns partition_channels(J, 2)[rank], computes its channel-block partial of the
    window channel sum (FP64) and its coil outputs, the partials are exchanged and
    summed in member order, the rho part of a dot product is counted once, and the
    assembled result equals the single-process apply_normal of the numpy
    restatement (oracle/nlinv_np.py; the device groups in group.cu follow the same
    contract through peer memory).
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist
        import bench
        from oracle import nlinv_np as o

        r, w, local = bench.dist_setup(world, backend="gloo")
        assert (r, w) == (rank, world)
        bench.barrier(w, local)
        bench.host_barrier(w)  # the N > 1 headline's host-side wait (gloo group)
        span = bench.max_over_ranks(10.0 * (rank + 1), w, local)
        value = bench.weak_scaling_value(w, 20, span)

        # channel decomposition contract
        G, J = 32, 5
        Gc = G // 4
        lay = o.Layout(G, Gc, J)
        rng = np.random.default_rng(7)
        rnd = lambda *sh: (rng.uniform(-1, 1, sh) + 1j * rng.uniform(-1, 1, sh)).astype(np.complex64)
        x, dx, P = rnd(lay.D), rnd(lay.D), rnd(G, G)
        winv = o.make_weights_inv(Gc, G)
        full = o.apply_normal(dx, o.StepCache(x, lay, P, winv))
        j0, j1 = o.partition_channels(J, w, cap=8)[r]
        sub = o.Layout(G, Gc, j1 - j0)
        pick = lambda e: np.concatenate([e[:G * G], e[G * G + j0 * Gc * Gc:G * G + j1 * Gc * Gc]])
        sc = o.StepCache(pick(x), sub, P, winv)
        drho, dchat = sub.split(pick(dx))
        part = np.zeros((G, G), np.complex128)
        out_chat = np.zeros((j1 - j0, Gc, Gc), np.complex64)
        for j in range(j1 - j0):  # the member's channels, in channel order
            cj = sc.coils[j]
            t = o.apply_W_inv(dchat[j], winv, G)
            t = ((cj * drho).astype(np.complex64) + (sc.rho * t).astype(np.complex64)).astype(np.complex64)
            t = o.toeplitz_apply(t, P)
            part += (np.conj(cj) * t).astype(np.complex64).astype(np.complex128)
            out_chat[j] = o.apply_W_invH((np.conj(sc.rho) * t).astype(np.complex64), winv, Gc)
        parts = [torch.zeros(2 * G * G, dtype=torch.float64) for _ in range(w)]
        dist.all_gather(parts, torch.from_numpy(part.view(np.float64).ravel().copy()))
        rho_sum = np.zeros((G, G), np.complex128)
        for p in parts:  # member order
            rho_sum += p.numpy().view(np.complex128).reshape(G, G)
        out_rho = rho_sum.astype(np.complex64)
        # <dx, out>: rho part once (member 0), chat parts from every member, member order
        loc = o.est_dot(dchat.ravel(), out_chat.ravel()).real + (o.est_dot(drho.ravel(), out_rho.ravel()).real
                                                                 if r == 0 else 0.0)
        dots = [torch.zeros(1, dtype=torch.float64) for _ in range(w)]
        dist.all_gather(dots, torch.tensor([loc], dtype=torch.float64))
        dot = sum(float(d.item()) for d in dots)
        chats = [torch.zeros(2 * J * Gc * Gc, dtype=torch.float32) for _ in range(w)]
        mine = np.zeros((J, Gc, Gc), np.complex64)
        mine[j0:j1] = out_chat
        dist.all_gather(chats, torch.from_numpy(mine.view(np.float32).ravel().copy()))
        assembled = np.zeros((J, Gc, Gc), np.complex64)
        for k, c in enumerate(chats):
            a0, a1 = o.partition_channels(J, w, cap=8)[k]
            assembled[a0:a1] = c.numpy().view(np.complex64).reshape(J, Gc, Gc)[a0:a1]
        frho, fchat = lay.split(full)
        err_rho = float(np.linalg.norm(out_rho - frho) / np.linalg.norm(frho))
        err_chat = float(np.linalg.norm(assembled - fchat) / np.linalg.norm(fchat))
        full_dot = o.est_dot(dx, full).real
        q.put((rank, span, value, (j0, j1), err_rho, err_chat, abs(dot - full_dot) / abs(full_dot)))
        dist.destroy_process_group()
    except Exception as e:  # surfaced by the parent
        q.put((rank, "error", repr(e)))


def test_two_rank_gloo_plumbing_and_channel_contract():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[1] != "error", r
    res.sort()
    assert [r[0] for r in res] == [0, 1]
    for rank, span, value, block, err_rho, err_chat, err_dot in res:
        assert span == 20.0  # max over ranks
        assert value == pytest.approx(2 * 20 / 0.020)
        assert err_rho < 1e-6 and err_chat == 0.0 and err_dot < 1e-9
    assert [r[3] for r in res] == [(0, 3), (3, 5)]
