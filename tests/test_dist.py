"""Host-side logic of the multi-GPU subtree sharding (-m "not gpu"), including a world_size-2 gloo run:
the shard plan partitions the sorted rows and the leaves exactly as the count-median tree does
(Fig. 6 line 1), and the NCCL id broadcast of Dist.from_torch hands every
rank the same 128-byte id."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1403_6015_b200.hodlr as hb
from paper_1403_6015_b200.dist import Dist


def tree_ranges(n, leaf):
    """Count-median tree written out independently of the library: kappa and node ranges by depth."""
    kappa = 0
    while leaf * 2 ** (kappa + 1) <= n:
        kappa += 1
    levels = [[(0, n)]]
    for _ in range(kappa):
        nxt = []
        for lo, hi in levels[-1]:
            half = (hi - lo + 1) // 2
            nxt += [(lo, lo + half), (lo + half, hi)]
        levels.append(nxt)
    return kappa, levels


@pytest.mark.parametrize("n,leaf,P", [(1 << 20, 128, 8), (1 << 20, 128, 2), (1000003, 100, 4), (131072, 64, 8),
                                      (2048, 64, 32), (777, 50, 8), (4096, 64, 1)])
def test_plan_partitions_rows_and_leaves(n, leaf, P):
    kappa, levels = tree_ranges(n, leaf)
    t = P.bit_length() - 1
    plans = [hb.hodlr_dist_plan(n, leaf, r, P) for r in range(P)]
    assert all(p["kappa"] == kappa and p["t"] == t for p in plans)
    assert [(p["row_lo"], p["row_hi"]) for p in plans] == levels[t]
    assert plans[0]["row_lo"] == 0 and plans[-1]["row_hi"] == n
    per = 2 ** (kappa - t)
    assert [(p["leaf_lo"], p["leaf_hi"]) for p in plans] == [(r * per, (r + 1) * per) for r in range(P)]
    # the leaves of rank r lie inside its rows
    for r, p in enumerate(plans):
        leaves = levels[kappa][p["leaf_lo"]:p["leaf_hi"]]
        assert leaves[0][0] == p["row_lo"] and leaves[-1][1] == p["row_hi"]


@pytest.mark.parametrize("n,leaf,P", [(1 << 10, 64, 3), (1 << 10, 64, 32), (100, 64, 2), (1 << 10, 64, 0)])
def test_plan_rejects_invalid_splits(n, leaf, P):
    with pytest.raises(hb.HodlrError) as e:
        hb.hodlr_dist_plan(n, leaf, 0, P)
    assert e.value.status == "EINVAL"


def _free_port():
    s = socket.socket(); s.bind(("127.0.0.1", 0)); p = s.getsockname()[1]; s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        n, leaf = 1 << 16, 128
        p = hb.hodlr_dist_plan(n, leaf, rank, ws)
        mine = torch.tensor([p["row_lo"], p["row_hi"], p["leaf_lo"], p["leaf_hi"]], dtype=torch.int64)
        allp = [torch.zeros(4, dtype=torch.int64) for _ in range(ws)]
        dist.all_gather(allp, mine)
        rows = [(int(a[0]), int(a[1])) for a in allp]
        ok_rows = rows[0][0] == 0 and rows[-1][1] == n and all(rows[i][1] == rows[i + 1][0] for i in range(ws - 1))
        d = Dist.from_torch()                           # rank 0 creates the ncclUniqueId, gloo broadcasts it
        ids = [None] * ws
        dist.all_gather_object(ids, d._id.raw)
        st = d.struct()
        q.put((rank, ok_rows, len(set(ids)) == 1 and len(ids[0]) == 128, st.rank, st.nranks, bool(st.nccl_unique_id),
               st.group is None))
    finally:
        dist.destroy_process_group()


def test_gloo_world_size_2():
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, (rank, ok_rows, same_id, srank, snr, has_id, no_group) in enumerate(res):
        assert rank == r and ok_rows and same_id and srank == r and snr == ws and has_id and no_group
