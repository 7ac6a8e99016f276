"""Multi-process host logic of the tile sharding on CPU with gloo,
world_size 2: the demand-driven queue hands every tile out exactly once, the in-flight
window never exceeds n_slots (SPEC.md:398's window invariant, via a null pipeline that
mimics hp_run_tiles' slot discipline), and the gathered table is the sorted union --
identical to a single-process run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1209_3332_b200.dist import (DistTileSource, TileQueue, aggregate_groups, gather_rows, table_digest,
                                       to_rows)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_rows(tid):
    rng = np.random.default_rng(tid)
    n = int(rng.integers(0, 5))
    lab = np.sort(rng.choice(10_000, size=n, replace=False)).astype(np.int32) + 1
    fl = (lab % 2).astype(np.int32)
    ft = rng.random((n, 36)).astype(np.float32)
    return lab, fl, ft


def _null_run(source, n_slots, inflight_log):
    """Stand-in for hp_run_tiles: round-robin slots, at most n_slots tiles in flight."""
    results, slots = {}, [None] * n_slots
    i = 0
    while True:
        if slots[i] is not None:
            tid = slots[i]
            results[tid] = _fake_rows(tid)
            slots[i] = None
        r = source()
        if r is None:
            for k in range(n_slots):
                if slots[k] is not None:
                    results[slots[k]] = _fake_rows(slots[k])
                    slots[k] = None
            return results
        slots[i] = r[2]
        inflight_log.append(sum(s is not None for s in slots))
        i = (i + 1) % n_slots


def _worker(rank, world, port, n_tiles, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q = TileQueue(n_tiles, block=3)
    pool = [torch.zeros((4, 4, 3), dtype=torch.uint8) for _ in range(5)]
    src = DistTileSource(q, lambda tid: pool[tid % len(pool)])
    log = []
    res = _null_run(src, n_slots=2, inflight_log=log)
    table = gather_rows(res)
    if rank == 0:
        out_q.put((sorted(src.taken), table_digest(table), len(table), max(log) if log else 0))
    else:
        out_q.put((sorted(src.taken), None, None, max(log) if log else 0))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_tiles", [0, 1, 37])
def test_queue_and_gather_world2(n_tiles):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_tiles, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    taken = sorted(t for o in outs for t in o[0])
    assert taken == list(range(n_tiles))                      # every tile exactly once
    assert all(o[3] <= 2 for o in outs)                        # window bound (n_slots = 2)
    digest = next(o[1] for o in outs if o[1] is not None)
    ref = {t: _fake_rows(t) for t in range(n_tiles)}
    assert digest == table_digest(to_rows(ref).sorted())       # sorted union = 1-process table


def test_rows_columns_and_merge():
    from paper_1209_3332_b200.dist import merge_tile_runs
    res = {7: _fake_rows(7), 3: _fake_rows(3), 11: _fake_rows(11)}
    rec = to_rows(res)
    assert list(rec.tile) == [3] * len(res[3][0]) + [7] * len(res[7][0]) + [11] * len(res[11][0])
    assert np.array_equal(rec.label[:len(res[3][0])], res[3][0])
    assert rec.feat.shape == (len(rec), 36)
    # two "ranks" holding interleaved tiles merge into the 1-process order
    a = to_rows({3: res[3], 11: res[11]})
    b = to_rows({7: res[7]})
    assert table_digest(merge_tile_runs([a, b])) == table_digest(rec)
    assert table_digest(merge_tile_runs([b, a])) == table_digest(rec.sorted())


def test_single_process_queue():
    q = TileQueue(10, block=4, store=None)
    blocks = []
    while (b := q.grab()) is not None:
        blocks.append(list(b))
    assert blocks == [[0, 1, 2, 3], [4, 5, 6, 7], [8, 9]]


class HostReducer:
    """Test stand-in for a Context's three aggregation kernels (hp_reduce_rows,
    hp_group_center, hp_group_std) on CPU tensors, so the gloo tests exercise the host logic
    of dist.aggregate_groups (two passes, two all-reduces) without a GPU.  The product has no
    host reducer."""

    @staticmethod
    def reduce_rows(feat, off, out, count):
        f, o = feat.numpy().astype(np.float64), off.numpy()
        for g in range(len(o) - 1):
            x = f[o[g]:o[g + 1]]
            out[g, :, 0] = torch.from_numpy(x.sum(axis=0))
            out[g, :, 1] = torch.from_numpy((x * x).sum(axis=0))
            count[g] = int(o[g + 1] - o[g])

    @staticmethod
    def group_center(feat, off, sums, count, mean_m2):
        f, o = feat.numpy().astype(np.float64), off.numpy()
        for g in range(len(o) - 1):
            n = int(count[g])
            m = sums[g, :, 0].numpy() / n if n else np.full(36, np.nan)
            mean_m2[g, :, 0] = torch.from_numpy(m)
            mean_m2[g, :, 1] = torch.from_numpy(((f[o[g]:o[g + 1]] - m) ** 2).sum(axis=0))

    @staticmethod
    def group_std(mean_m2, count, mean, std):
        for g in range(count.shape[0]):
            n = int(count[g])
            mean[g] = mean_m2[g, :, 0]
            std[g] = torch.sqrt(mean_m2[g, :, 1] / n) if n else float("nan")


def _agg_worker(rank, world, port, n_tiles, out_q, empty_rank=-1):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # disjoint tiles; with empty_rank set, that rank holds no rows at all (it must
    # still join both all-reduces instead of failing and hanging the others)
    mine = {t: _fake_rows(t) for t in range(n_tiles)
            if (t % world == rank if empty_rank < 0 else rank != empty_rank)}
    cnt, mean, std = aggregate_groups(to_rows(mine), lambda tile: tile // 5, (n_tiles + 4) // 5, HostReducer())
    out_q.put((rank, cnt, mean, std))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("empty_rank", [-1, 1])
def test_aggregate_groups_world2(empty_rank):
    """SURVEY NEXT-4 host logic: per-rank partial sums, all-reduce, per-rank centred sums,
    all-reduce == the oracle's per-group mean / population std over the union of the rows
    (also when one rank holds no rows)."""
    import oracle
    n_tiles = 23
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agg_worker, args=(r, 2, port, n_tiles, q, empty_rank)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=120) for _ in procs], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = to_rows({t: _fake_rows(t) for t in range(n_tiles)})
    G = (n_tiles + 4) // 5
    off = np.searchsorted(ref.tile // 5, np.arange(G + 1))
    rc, rm, rs = oracle.aggregate(ref.feat, off)
    for _, cnt, mean, std in outs:
        assert np.array_equal(cnt, rc)
        assert np.allclose(mean, rm, rtol=1e-12, atol=1e-12, equal_nan=True)
        assert np.allclose(std, rs, rtol=1e-9, atol=1e-12, equal_nan=True)



def test_bind_to_gpu_numa_without_nvml_is_a_no_op():
    """Without a GPU/NVML the binding helper changes nothing and says so (returns None)."""
    import os

    import torch
    from paper_1209_3332_b200.dist import bind_to_gpu_numa
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    before = os.sched_getaffinity(0)
    assert bind_to_gpu_numa(0) is None
    assert os.sched_getaffinity(0) == before
