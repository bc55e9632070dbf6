"""Host-side logic of the multi-rank (row-partitioned) path, on CPU with torch.distributed
gloo, world_size 2 and 3: the CSR halo plans computed independently by each rank (through
the C ABI's refine_halo_plan, the routine the multi-rank init uses) must pair up -- every
segment a rank sends is exactly a segment its peer receives -- and each rank's receive
segments must cover exactly the columns its rows reference but do not own; the ncclUniqueId
bootstrap (refine_nccl_id on rank 0, broadcast over the process group) must reach every rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partition(n, world, k):
    blk = n // world
    rb = [0 if r == 0 else n - blk * (world - r) for r in range(world)]
    re = [n - blk * (world - r - 1) for r in range(world)]
    assert re[0] - rb[0] >= k
    return rb, re


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2602_23778_b200 as pkg
        p = synth.small_laplacian((23, 17, 9), (1.0, 1.13, 1.29), 4)
        rp, ci = p.row_ptr.numpy(), p.col_idx.numpy()
        rb, re = _partition(p.n, world, p.k)
        # each rank knows only its own rows: column range of its CSR rows, then all-gather
        mine = ci[rp[rb[rank]]:rp[re[rank]]]
        info = torch.tensor([rb[rank], re[rank], min(mine.min(), rb[rank]), max(mine.max(), re[rank] - 1)],
                            dtype=torch.int64)
        allinfo = [torch.zeros(4, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allinfo, info)
        a = torch.stack(allinfo).numpy()
        send, recv, hrows = pkg.refine_halo_plan(world, rank, a[:, 0], a[:, 1], a[:, 2], a[:, 3])
        # the rows this rank needs but does not own are exactly the halo
        need = np.unique(mine)
        need = need[(need < rb[rank]) | (need >= re[rank])]
        got = np.concatenate([np.arange(r, r + c) for (_, r, c, _) in recv]) if recv else np.zeros(0, np.int64)
        lo, hi = a[rank, 2], a[rank, 3]
        halo_rows = np.concatenate([np.arange(lo, rb[rank]), np.arange(re[rank], hi + 1)])
        assert np.array_equal(np.sort(got), halo_rows), "recv segments != halo range"
        assert set(need.tolist()) <= set(got.tolist()), "a referenced column is not received"
        assert hrows == len(halo_rows)
        for (peer, r0, cnt, off) in recv:       # halo offsets: [lo, rb) then [re, hi]
            exp = r0 - lo if r0 < rb[rank] else (rb[rank] - lo) + (r0 - re[rank])
            assert off == exp and rb[peer] <= r0 and r0 + cnt <= re[peer]
        for (peer, r0, cnt, off) in send:
            assert off == r0 - rb[rank] and rb[rank] <= r0 and r0 + cnt <= re[rank]
        # pair every send with the peer's receive
        plans = [None] * world
        dist.all_gather_object(plans, (send, recv))
        for (peer, r0, cnt, _) in send:
            assert any(pr == rank and rr == r0 and rc == cnt for (pr, rr, rc, _) in plans[peer][1])
        for (peer, r0, cnt, _) in recv:
            assert any(pr == rank and rr == r0 and rc == cnt for (pr, rr, rc, _) in plans[peer][0])
        # ncclUniqueId bootstrap over the process group (skipped if NCCL cannot be loaded here)
        ok = torch.zeros(1)
        buf = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            try:
                buf = torch.frombuffer(bytearray(pkg.refine_nccl_id()), dtype=torch.uint8).clone()
                ok[0] = 1
            except Exception:
                ok[0] = 0
        dist.broadcast(ok, 0)
        dist.broadcast(buf, 0)
        if ok[0] == 1:
            ids = [torch.zeros(128, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(ids, buf)
            assert all(torch.equal(ids[0], x) for x in ids) and int(ids[0].sum()) != 0
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_plans_pair_up_gloo(world):
    from paper_2602_23778_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(msg == "ok" for _, msg in res), res


def test_halo_plan_single_rank_is_empty():
    import paper_2602_23778_b200 as pkg
    send, recv, hr = pkg.refine_halo_plan(1, 0, [0], [100], [0], [99])
    assert send == [] and recv == [] and hr == 0
