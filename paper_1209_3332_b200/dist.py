"""Multi-GPU plumbing for the tile pipeline.

Tiles are independent and the paper replicates the whole pipeline per
worker, so the data path has no exchange step:

* ``TileQueue`` -- demand-driven dispatch: ranks pull blocks of
  consecutive tile ids from one shared counter (an atomic ``add`` on the process group's
  key-value store), so faster GPUs simply take more tiles.
* ``DistTileSource`` -- feeds ``Context.run_tiles`` (hp_run_tiles: per-slot H2D / compute /
  D2H streams, at most n_slots tiles in flight = the paper's window).
* ``gather_rows`` -- the one collective: at the end, every rank's feature rows go to rank 0
  (all_gather of counts, then a padded all_gather_into_tensor of packed rows -- NCCL over
  NVLink on GPUs, gloo on CPU), sorted by (tile_id, label) so the table is identical for
  any number of GPUs.

torch.distributed is plumbing here; the pixels never leave the GPU that processes them.
"""
from __future__ import annotations

import hashlib

import numpy as np

NFEAT = 34
ROW_BYTES = 8 + 4 + 4 + 4 * NFEAT  # tile_id i64, label i32, flags i32, feat f32[34]


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


ROW_DTYPE = np.dtype([("tile", "<i8"), ("label", "<i4"), ("flags", "<i4"), ("feat", "<f4", (NFEAT,))])


def pack_rows(results: dict) -> np.ndarray:
    """{tile_id: (label[n], flags[n], feat[n, 34])} -> uint8 [N, ROW_BYTES] (tile order)."""
    tids = sorted(results)
    counts = [len(results[t][0]) for t in tids]
    total = int(sum(counts))
    rec = np.empty(total, dtype=ROW_DTYPE)
    if total:
        rec["tile"] = np.repeat(np.asarray(tids, np.int64), counts)
        rec["label"] = np.concatenate([results[t][0] for t in tids])
        rec["flags"] = np.concatenate([results[t][1] for t in tids])
        rec["feat"] = np.concatenate([np.asarray(results[t][2], np.float32).reshape(-1, NFEAT) for t in tids])
    return rec.view(np.uint8).reshape(total, ROW_BYTES)


def unpack_rows(buf: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(buf).view(ROW_DTYPE).reshape(-1)


def gather_rows(results: dict, device=None):
    """Gather every rank's packed rows on rank 0 (sorted by tile, label); None elsewhere."""
    import torch
    import torch.distributed as dist
    local = pack_rows(results)
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return unpack_rows(local)  # pack_rows emits tile order; rows within a tile are label order
    world = dist.get_world_size()
    dev = device if device is not None else torch.device("cpu")
    cnt = torch.tensor([local.shape[0]], dtype=torch.int64, device=dev)
    counts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(counts, cnt)
    counts = [int(c.item()) for c in counts]
    mx = max(counts) if counts else 0
    pad = torch.zeros((mx, ROW_BYTES), dtype=torch.uint8, device=dev)
    if local.shape[0]:
        pad[:local.shape[0]] = torch.from_numpy(local).to(dev)
    out = torch.zeros((world * mx, ROW_BYTES), dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(out, pad)
    if dist.get_rank() != 0:
        return None
    allb = out.cpu().numpy().reshape(world, mx, ROW_BYTES)
    rows = np.concatenate([allb[r, :counts[r]] for r in range(world)], axis=0)
    rec = unpack_rows(rows)
    return rec[np.lexsort((rec["label"], rec["tile"]))]


def table_digest(rec: np.ndarray) -> str:
    """Order-independent content digest of a gathered (sorted) table."""
    return hashlib.sha256(np.ascontiguousarray(rec).view(np.uint8).tobytes()).hexdigest()[:16]
