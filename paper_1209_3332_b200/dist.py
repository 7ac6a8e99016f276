"""Multi-GPU plumbing for the tile pipeline.

Tiles are independent and the paper replicates the whole pipeline per
worker, so the data path has no exchange step:

* ``TileQueue`` -- demand-driven dispatch: ranks pull blocks of
  consecutive tile ids from one shared counter (an atomic ``add`` on the process group's
  key-value store), so faster GPUs simply take more tiles.
* ``DistTileSource`` -- feeds ``Context.run_tiles`` (hp_run_tiles: per-slot H2D / compute /
  D2H streams, at most n_slots tiles in flight = the paper's window).
* ``RowArena`` / ``gather_rows_device`` -- the one collective: rows stay on the GPU in an
  hp_row_arena during the run; at the end every rank sends its rows to rank 0 device to
  device (NCCL point-to-point over NVLink; gloo on CPU), where a stable sort by tile id gives
  the (tile_id, label) order, so the table is identical for any number of GPUs.

torch.distributed is plumbing here; the pixels never leave the GPU that processes them.
"""
from __future__ import annotations

import hashlib

import numpy as np

NFEAT = 36
ROW_BYTES = 8 + 4 + 4 + 4 * NFEAT  # tile_id i64, label i32, flags i32, feat f32[36]


def bind_to_gpu_numa(device: int) -> list | None:
    """Pin this process to the CPU cores nearest GPU `device` (NVML's CPU affinity), so the
    pinned host buffers it allocates afterwards (first touch) and its feeder thread sit on the
    GPU's NUMA node: host->device copies then never cross the socket link.  Returns the cores,
    or None when NVML is unavailable.  Call before allocating pinned memory."""
    import os
    try:
        import pynvml
        pynvml.nvmlInit()
        try:
            vis = [v.strip() for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
            if device < len(vis) and vis[device].startswith("GPU-"):
                h = pynvml.nvmlDeviceGetHandleByUUID(vis[device])
            else:
                phys = int(vis[device]) if device < len(vis) else device
                h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        finally:
            pynvml.nvmlShutdown()
    except Exception:  # noqa: BLE001 -- no NVML (CPU tests): leave the affinity alone
        return None
    cores = [64 * i + b for i, wd in enumerate(words) for b in range(64) if (wd >> b) & 1]
    cores = [c for c in cores if c < (os.cpu_count() or 0)]
    if not cores:
        return None
    try:
        os.sched_setaffinity(0, cores)
    except OSError:
        return None
    return cores


def _default_store():
    import torch.distributed as dist
    from torch.distributed import distributed_c10d as c10d
    if not dist.is_initialized():
        return None
    return c10d._get_default_store()


class TileQueue:
    """Shared tile-id dispenser.  ``grab()`` returns the next block of ids or None."""

    def __init__(self, n_tiles: int, block: int = 4, store=None, key: str = "hp/next_tile"):
        self.n_tiles = int(n_tiles)
        self.block = max(1, int(block))
        self.store = store if store is not None else _default_store()
        self.key = key
        self._local = 0  # single-process fallback

    def grab(self):
        if self.store is None:
            start = self._local
            self._local += self.block
        else:
            start = int(self.store.add(self.key, self.block)) - self.block
        if start >= self.n_tiles:
            return None
        return range(start, min(start + self.block, self.n_tiles))


class DistTileSource:
    """Iterator of (host_ptr, pitch, tile_id) for Context.run_tiles, pulling from a queue.

    ``get_tile(tile_id)`` must return a pinned host uint8 tensor [H, W, 3] that stays alive
    until the tile's result has been delivered (the pool tensors are kept by the caller)."""

    def __init__(self, queue: TileQueue, get_tile):
        self.queue = queue
        self.get_tile = get_tile
        self._ids = iter(())
        self.taken = []

    def __call__(self):
        while True:
            try:
                tid = next(self._ids)
                break
            except StopIteration:
                blk = self.queue.grab()
                if blk is None:
                    return None
                self._ids = iter(blk)
        t = self.get_tile(tid)
        self.taken.append(tid)
        return t.data_ptr(), t.stride(0) * t.element_size(), tid


class Rows:
    """A feature table in columns: tile id, label, flags, 36 features per object row."""

    __slots__ = ("tile", "label", "flags", "feat")

    def __init__(self, tile, label, flags, feat):
        self.tile = np.ascontiguousarray(tile, dtype=np.int64)
        self.label = np.ascontiguousarray(label, dtype=np.int32)
        self.flags = np.ascontiguousarray(flags, dtype=np.int32)
        self.feat = np.ascontiguousarray(feat, dtype=np.float32).reshape(-1, NFEAT)

    def __len__(self):
        return int(self.tile.shape[0])

    def take(self, a, b):
        return Rows(self.tile[a:b], self.label[a:b], self.flags[a:b], self.feat[a:b])

    @staticmethod
    def concat(parts):
        if not parts:
            return Rows(np.empty(0, np.int64), np.empty(0, np.int32), np.empty(0, np.int32),
                        np.empty((0, NFEAT), np.float32))
        return Rows(np.concatenate([p.tile for p in parts]), np.concatenate([p.label for p in parts]),
                    np.concatenate([p.flags for p in parts]), np.concatenate([p.feat for p in parts]))

    def sorted(self):
        """(tile, label) order -- the canonical table order (reading C14)."""
        o = np.lexsort((self.label, self.tile))
        return Rows(self.tile[o], self.label[o], self.flags[o], self.feat[o])


def to_rows(results: dict) -> Rows:
    """{tile_id: (label[n], flags[n], feat[n, 36])} -> Rows in tile order (rows of a tile in
    the order given: hp_run_tiles delivers them by ascending label)."""
    tids = sorted(results)
    counts = [len(results[t][0]) for t in tids]
    if not tids or sum(counts) == 0:
        return Rows.concat([])
    return Rows(np.repeat(np.asarray(tids, np.int64), counts),
                np.concatenate([results[t][0] for t in tids]),
                np.concatenate([results[t][1] for t in tids]),
                np.concatenate([np.asarray(results[t][2], np.float32).reshape(-1, NFEAT) for t in tids]))


_FIELDS = (("tile", np.int64, 8), ("label", np.int32, 4), ("flags", np.int32, 4), ("feat", np.float32, 4 * NFEAT))


class DeviceRows:
    """A feature table resident in device memory (torch tensors): tile i64[n], label i32[n],
    flags i32[n], feat f32[n, 36] -- e.g. the first ``cursor`` rows of an hp_row_arena."""

    __slots__ = ("tile", "label", "flags", "feat")

    def __init__(self, tile, label, flags, feat):
        self.tile, self.label, self.flags, self.feat = tile, label, flags, feat

    def __len__(self):
        return int(self.tile.shape[0])

    def to_host(self) -> Rows:
        return Rows(self.tile.cpu().numpy(), self.label.cpu().numpy(), self.flags.cpu().numpy(),
                    self.feat.cpu().numpy())

    @staticmethod
    def from_host(rows: Rows, device):
        import torch
        return DeviceRows(*(torch.from_numpy(np.ascontiguousarray(getattr(rows, n))).to(device)
                            for n in ("tile", "label", "flags", "feat")))


class RowArena:
    """Device buffers of an hp_row_arena (hp.h): hp_run_tiles appends every tile's rows here,
    so the rows never leave the GPU; ``arena`` is the tuple Context.run_tiles takes."""

    def __init__(self, capacity: int, device):
        import torch
        self.capacity = int(capacity)
        self.tile = torch.empty(self.capacity, dtype=torch.int64, device=device)
        self.label = torch.empty(self.capacity, dtype=torch.int32, device=device)
        self.flags = torch.empty(self.capacity, dtype=torch.int32, device=device)
        self.feat = torch.empty((self.capacity, NFEAT), dtype=torch.float32, device=device)
        self.cursor = torch.zeros(1, dtype=torch.int64, device=device)

    @property
    def arena(self):
        return (self.tile.data_ptr(), self.label.data_ptr(), self.flags.data_ptr(), self.feat.data_ptr(),
                self.capacity, self.cursor.data_ptr())

    def rows(self) -> DeviceRows:
        """The rows appended so far (reads the cursor: one device synchronisation)."""
        n = min(int(self.cursor.item()), self.capacity)
        return DeviceRows(self.tile[:n], self.label[:n], self.flags[:n], self.feat[:n])


def gather_rows_device(rows: DeviceRows, device=None, stats: dict | None = None):
    """The end-of-run gather: every rank's device-resident rows go to rank 0
    only, device to device (NCCL point-to-point over NVLink on GPUs; gloo on CPU) -- no host
    round trip and no all-gather to every rank.  Rank 0 returns the merged table in
    (tile, label) order as DeviceRows, the other ranks None.  Each tile's rows are one
    contiguous run in label order on one rank (hp_run_tiles delivers a tile's rows at once),
    so a stable sort by tile id gives the canonical order for any number of GPUs.  With
    ``stats`` (a dict) the transfer and the merge are timed separately (synchronising)."""
    import time

    import torch
    import torch.distributed as dist
    dev = device if device is not None else rows.tile.device
    t0 = time.perf_counter()
    if not dist.is_initialized() or dist.get_world_size() == 1:
        parts = [rows]
    else:
        world, rank = dist.get_world_size(), dist.get_rank()
        cnt = torch.tensor([len(rows)], dtype=torch.int64, device=dev)
        counts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
        dist.all_gather(counts, cnt)           # 8 bytes per rank
        counts = [int(c.item()) for c in counts]
        cols = ("tile", "label", "flags", "feat")
        if rank != 0:
            ops = [dist.P2POp(dist.isend, getattr(rows, c).contiguous(), 0) for c in cols] if counts[rank] else []
            for w in (dist.batch_isend_irecv(ops) if ops else []):
                w.wait()
            return None
        parts = [rows]
        ops = []
        for r in range(1, world):
            n = counts[r]
            if n == 0:
                continue
            part = DeviceRows(torch.empty(n, dtype=torch.int64, device=dev), torch.empty(n, dtype=torch.int32, device=dev),
                              torch.empty(n, dtype=torch.int32, device=dev),
                              torch.empty((n, NFEAT), dtype=torch.float32, device=dev))
            ops += [dist.P2POp(dist.irecv, getattr(part, c), r) for c in cols]
            parts.append(part)
        for w in (dist.batch_isend_irecv(ops) if ops else []):
            w.wait()
    on_gpu = torch.device(dev).type == "cuda"
    if stats is not None:
        if on_gpu:
            torch.cuda.synchronize(dev)
        stats["transfer_s"] = time.perf_counter() - t0
        stats["received_bytes"] = sum(len(p) for p in parts[1:]) * ROW_BYTES
    t1 = time.perf_counter()
    tile = torch.cat([p.tile for p in parts])
    order = torch.argsort(tile, stable=True)
    out = DeviceRows(tile[order], torch.cat([p.label for p in parts])[order],
                     torch.cat([p.flags for p in parts])[order], torch.cat([p.feat for p in parts])[order])
    if stats is not None:
        if on_gpu:
            torch.cuda.synchronize(dev)
        stats["merge_s"] = time.perf_counter() - t1
    return out


def sort_rows(rows: DeviceRows) -> DeviceRows:
    """(tile, label) order of one rank's device rows (a stable sort by tile id: each tile's
    rows are one label-ordered run)."""
    import torch
    order = torch.argsort(rows.tile, stable=True)
    return DeviceRows(rows.tile[order], rows.label[order], rows.flags[order], rows.feat[order])


def gather_rows(results: dict, device=None):
    """Gather host-delivered rows ({tile_id: (label, flags, feat)}, the sink callback's output)
    on rank 0 in (tile, label) order through gather_rows_device; None on other ranks."""
    import torch
    dev = device if device is not None else torch.device("cpu")
    out = gather_rows_device(DeviceRows.from_host(to_rows(results), dev), dev)
    return None if out is None else out.to_host()


def merge_tile_runs(parts) -> Rows:
    """Merge per-rank tables into (tile, label) order.  Each rank's table is already in that
    order and a tile belongs to one rank, so sorting the per-tile runs and concatenating them
    is enough -- O(rows) copying instead of sorting every row."""
    runs = []
    for r, rec in enumerate(parts):
        if len(rec) == 0:
            continue
        t = rec.tile
        starts = np.flatnonzero(np.r_[True, t[1:] != t[:-1]])
        ends = np.r_[starts[1:], len(t)]
        runs.extend((int(t[a]), r, int(a), int(b)) for a, b in zip(starts, ends))
    runs.sort()
    return Rows.concat([parts[r].take(a, b) for _, r, a, b in runs])


def table_digest(rows: Rows) -> str:
    """Content digest of a table (column by column)."""
    h = hashlib.sha256()
    for name, _, _ in _FIELDS:
        h.update(np.ascontiguousarray(getattr(rows, name)).view(np.uint8).tobytes())
    return h.hexdigest()[:16]


def group_offsets(rows: Rows, group_of_tile, n_groups: int) -> np.ndarray:
    """Row offsets of each group (int64[n_groups + 1]) in a tile-ordered table, for a group
    id that is non-decreasing in the tile id (e.g. slide = tile // tiles_per_slide)."""
    gid = np.asarray(group_of_tile(rows.tile), np.int64)
    if len(gid) and (np.any(np.diff(gid) < 0) or gid[0] < 0 or gid[-1] >= n_groups):
        raise ValueError("group ids must be non-decreasing in the table order and in [0, n_groups)")
    return np.searchsorted(gid, np.arange(n_groups + 1), side="left").astype(np.int64)


def aggregate_groups(rows: Rows, group_of_tile, n_groups: int, reduce, device=None):
    """Per-image (per-group) feature aggregation: the mean
    and population standard deviation of every feature over each group's object rows, in two
    device passes with one all-reduce after each (NCCL on GPUs, gloo on CPU):

    1. ``reduce.reduce_rows`` (hp_reduce_rows): per-rank segmented sums and row counts;
       all_reduce(SUM) gives the totals, hence every group's mean.
    2. ``reduce.group_center`` (hp_group_center): per-rank sums of squared deviations from
       that mean; all_reduce(SUM); ``reduce.group_std`` (hp_group_std) finishes std on the
       device.

    ``reduce`` is a Context (the device kernels); there is no host fallback.  A rank holding
    no rows still takes part in both all-reduces (its partial sums are zero).  Returns
    (count [G], mean [G, 36], std [G, 36]) as numpy (int64, float64, float64); NaN for an
    empty group."""
    import torch
    import torch.distributed as dist
    if reduce is None or not all(hasattr(reduce, m) for m in ("reduce_rows", "group_center", "group_std")):
        raise TypeError("aggregate_groups needs a Context (hp_reduce_rows / hp_group_center / hp_group_std)")
    dev = device if device is not None else torch.device("cpu")
    multi = dist.is_initialized() and dist.get_world_size() > 1
    if isinstance(rows, DeviceRows):  # rows already on the device (e.g. a RowArena, sorted)
        gid = group_of_tile(rows.tile)
        if len(rows) and (bool((gid[1:] < gid[:-1]).any()) or int(gid[0]) < 0 or int(gid[-1]) >= n_groups):
            raise ValueError("group ids must be non-decreasing in the table order and in [0, n_groups)")
        feat_t = rows.feat.contiguous()
        off_t = torch.searchsorted(gid.contiguous(), torch.arange(n_groups + 1, dtype=gid.dtype, device=gid.device))
    else:
        off = group_offsets(rows, group_of_tile, n_groups)
        feat_t = torch.from_numpy(np.ascontiguousarray(rows.feat)).to(dev)
        off_t = torch.from_numpy(off).to(dev)
    sums_t = torch.zeros((n_groups, NFEAT, 2), dtype=torch.float64, device=dev)
    cnt_t = torch.zeros(n_groups, dtype=torch.int64, device=dev)
    mm2_t = torch.zeros((n_groups, NFEAT, 2), dtype=torch.float64, device=dev)
    mean_t = torch.zeros((n_groups, NFEAT), dtype=torch.float64, device=dev)
    std_t = torch.zeros((n_groups, NFEAT), dtype=torch.float64, device=dev)
    if n_groups:
        reduce.reduce_rows(feat_t, off_t, sums_t, cnt_t)
    if multi:
        dist.all_reduce(sums_t, op=dist.ReduceOp.SUM)
        dist.all_reduce(cnt_t, op=dist.ReduceOp.SUM)
    if n_groups:
        reduce.group_center(feat_t, off_t, sums_t, cnt_t, mm2_t)
    if multi:
        # only the m2 half is additive; the mean half is identical on every rank
        m2 = mm2_t[:, :, 1].contiguous()
        dist.all_reduce(m2, op=dist.ReduceOp.SUM)
        mm2_t[:, :, 1] = m2
    if n_groups:
        reduce.group_std(mm2_t, cnt_t, mean_t, std_t)
    return cnt_t.cpu().numpy(), mean_t.cpu().numpy(), std_t.cpu().numpy()
