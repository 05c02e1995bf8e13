"""Multi-process (gloo, world_size 2/3) checks of the row partition and exchange."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2211_15082_b200.parallel import RowExchange, edge_balanced_ranges


def test_edge_balanced_ranges_cover_once_and_balance():
    rng = np.random.default_rng(0)
    degs = rng.zipf(2.0, size=10000).clip(max=3000)
    indptr = np.zeros(10001, dtype=np.int64)
    np.cumsum(degs, out=indptr[1:])
    for parts in (1, 2, 3, 4, 8):
        cuts = edge_balanced_ranges(indptr, parts)
        assert cuts[0] == 0 and cuts[-1] == 10000 and np.all(np.diff(cuts) >= 0)
        cost = np.diff(indptr + np.arange(10001))
        loads = [cost[cuts[k]:cuts[k + 1]].sum() for k in range(parts)]
        assert max(loads) <= cost.sum() / parts + cost.max()


def test_edge_balanced_ranges_degenerate():
    assert edge_balanced_ranges(np.zeros(1, dtype=np.int64), 4).tolist() == [0, 0, 0, 0, 0]
    assert edge_balanced_ranges(np.array([0, 5]), 2).tolist()[-1] == 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, dim, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    indptr = np.arange(n + 1, dtype=np.int64) * 3
    cuts = edge_balanced_ranges(indptr, world)
    ex = RowExchange(cuts, rank, world)
    data = torch.full((n, dim), -1.0)
    lo, hi = ex.row_range
    # each rank "computes" its rows: value = row id * 10 + column
    rows = torch.arange(lo, hi, dtype=torch.float32)[:, None] * 10 + torch.arange(dim)[None, :]
    data[lo:hi] = rows
    ex.exchange_tensor(data)
    want = torch.arange(n, dtype=torch.float32)[:, None] * 10 + torch.arange(dim)[None, :]
    result_q.put((rank, bool(torch.equal(data, want)), ex.bytes_sent, (lo, hi)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 37, 5, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _, _ in results)
    covered = sorted(r for _, _, _, r in results)
    assert covered[0][0] == 0 and covered[-1][1] == 37
    assert sum(b for _, _, b, _ in results) == 37 * 5 * 4


class _Store:
    def __init__(self, data):
        self.data = data


class _FakeSchedule:
    def __init__(self):
        from types import SimpleNamespace

        self.model_output = SimpleNamespace(key="out")
        self.drop_after = {"b1.h": 2}


class _FakeEngine:
    """Just what RowExchange reads: stores, schedule, users, transform_first."""

    def __init__(self, data):
        self.stores = {"b1.h": _Store(data)}
        self.schedule = _FakeSchedule()
        self.users = {"h": ["conv2"]}

    def transform_first(self, op):
        return False


def _progress_worker(rank, world, port, n, dim, result_q):
    from types import SimpleNamespace

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    indptr = np.arange(n + 1, dtype=np.int64) * 3
    cuts = edge_balanced_ranges(indptr, world)
    ex = RowExchange(cuts, rank, world, chunks=3)
    data = torch.full((n, dim), -1.0)
    eng = _FakeEngine(data)
    blk = SimpleNamespace(block_id=1, outputs=["h"], op_ids=["conv1", "h"])
    lo, hi = ex.row_range
    # rows are computed in batches of uneven size; progress after each batch
    step = max(1, (hi - lo) // 4 + rank)
    for s in range(lo, hi, step):
        e = min(hi, s + step)
        data[s:e] = torch.arange(s, e, dtype=torch.float32)[:, None] * 10 + torch.arange(dim)
        ex.progress(eng, blk, e)
    ex(eng, blk)
    want = torch.arange(n, dtype=torch.float32)[:, None] * 10 + torch.arange(dim)[None, :]
    result_q.put((rank, bool(torch.equal(data, want)), ex.bytes_sent))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_exchange_overlapped_pieces_gloo(world):
    """progress() posts finished pieces as batches complete (same order on every
    rank even though the ranks' batches differ); the block end completes it."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_progress_worker, args=(r, world, port, 41, 3, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in results)
    assert sum(b for _, _, b in results) == 41 * 3 * 4


def test_piece_bounds_cut_the_rank_range():
    """The engine cuts its launches at piece_bounds(), so each piece can be
    broadcast while the next computes; the bounds tile this rank's range."""
    from paper_2211_15082_b200.parallel import RowExchange

    ex = RowExchange(np.array([0, 10, 25]), rank=1, world=2, chunks=4)
    assert ex.piece_bounds() == [13, 17, 21, 25]
    assert [ex._piece(1, c) for c in range(4)] == [(10, 13), (13, 17), (17, 21), (21, 25)]
    ex0 = RowExchange(np.array([0, 10, 25]), rank=0, world=2, chunks=3)
    assert ex0.piece_bounds() == [3, 6, 10]


def _random_csc(n, e, seed):
    rng = np.random.default_rng(seed)
    dst = np.sort(rng.integers(0, n, size=e))
    src = rng.integers(0, n, size=e)
    indptr = np.concatenate([[0], np.cumsum(np.bincount(dst, minlength=n))]).astype(np.int64)
    return indptr, src.astype(np.int64)


def test_halo_plan_lists_exactly_the_remote_sources():
    """recv[k] = the distinct sources in rank k's range that this rank's slice reads;
    send[j] = what rank j's slice reads from this rank (the transpose)."""
    from paper_2211_15082_b200.parallel import HaloPlan

    indptr, src = _random_csc(300, 2000, 5)
    cuts = edge_balanced_ranges(indptr, 3)
    idx = torch.from_numpy(src).to(torch.int32)
    plans = [HaloPlan(indptr, idx, cuts, r) for r in range(3)]
    for j in range(3):
        mine = set(src[indptr[cuts[j]]:indptr[cuts[j + 1]]].tolist())
        for k in range(3):
            want = sorted(u for u in mine if cuts[k] <= u < cuts[k + 1]) if k != j else []
            assert plans[j].recv[k].tolist() == want
            assert plans[k].send[j].tolist() == want
    assert 0.0 < plans[0].fraction(300) <= 1.0


def _halo_worker(rank, world, port, n, e, dim, result_q):
    from types import SimpleNamespace

    from paper_2211_15082_b200.parallel import HaloPlan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    indptr, src = _random_csc(n, e, 9)
    cuts = edge_balanced_ranges(indptr, world)
    plan = HaloPlan(indptr, torch.from_numpy(src).to(torch.int32), cuts, rank)
    ex = RowExchange(cuts, rank, world, halo=plan)
    data = torch.full((n, dim), -1.0)
    lo, hi = ex.row_range
    want = torch.arange(n, dtype=torch.float32)[:, None] * 10 + torch.arange(dim)[None, :]
    data[lo:hi] = want[lo:hi]
    eng = _FakeEngine(data)
    blk = SimpleNamespace(block_id=1, outputs=["h"], op_ids=["conv1", "h"])
    ex.progress(eng, blk, hi)          # halo mode: nothing posted before the block end
    ex(eng, blk)
    read = np.unique(src[indptr[lo]:indptr[hi]])
    rows_ok = bool(torch.equal(data[read], want[read])) and bool(torch.equal(data[lo:hi], want[lo:hi]))
    untouched = np.setdiff1d(np.arange(n), np.concatenate([read, np.arange(lo, hi)]))
    stale_ok = bool(torch.all(data[untouched] == -1.0))
    # the model output is replicated in full whatever the mode
    full = torch.full((n, dim), -1.0)
    full[lo:hi] = want[lo:hi]
    ex.replicate_tensor(full)
    result_q.put((rank, rows_ok, stale_ok, bool(torch.equal(full, want)), ex.bytes_sent,
                  sum(plan.send_counts) * dim * 4))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_gloo(world):
    """Halo mode: every row a rank's slice reads (and its own rows) is exact after
    the exchange, rows nobody reads stay untouched, only the planned rows move,
    and replicate_tensor still delivers every row."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, 157, 300, 4, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, rows_ok, stale_ok, full_ok, sent, planned in results:
        assert rows_ok and stale_ok and full_ok, rank
        assert sent >= planned
