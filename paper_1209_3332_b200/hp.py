"""Thin ctypes binding of libhp (include/hp.h).  Argument marshalling only: every step of
the pipeline runs in the library's sm_100a kernels.  torch is used for device memory and
streams.  There is no fallback: if libhp.so is missing or the device is not a B200, the
calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("HP_SO", os.path.join(_HERE, "libhp.so"))

NFEAT = 36
FLAG_RBC_HI, FLAG_RBC_LO, FLAG_R_GT_B, FLAG_BG = 1, 2, 4, 8
OBJ_TOUCHES_BORDER = 1
FEATURE_NAMES = [
    "area", "perimeter", "centroid_x", "centroid_y", "bbox_w", "bbox_h", "major", "minor",
    "eccentricity", "orientation", "eqdiam", "compactness", "extent",
    "int_mean", "int_std", "int_min", "int_max", "int_median", "int_skew", "int_kurt",
    "int_entropy", "int_energy",
    "grad_mean", "grad_std", "grad_skew", "grad_kurt",
    "glcm_asm", "glcm_contrast", "glcm_correlation", "glcm_homogeneity", "glcm_entropy",
    "glcm_shade", "glcm_prominence", "glcm_maxprob",
    "edge_count", "edge_frac",
]
assert len(FEATURE_NAMES) == NFEAT

STAGES = ["CD", "RBC", "OPEN", "RECON", "AREA", "FILL", "EDT", "MARKERS", "WATERSHED",
          "BWLABEL", "FEATURES", "IWPP_RAW", "CCL8", "CCL4", "RECON_F32", "CANNY",
          "AREA_TOPHAT", "FILL_COMP", "COMPONENTS"]
STAGE = {n: i for i, n in enumerate(STAGES)}
STATUS = {0: "ok", 1: "invalid argument", 2: "CUDA error", 3: "out of memory",
          4: "object capacity exceeded", 5: "unsupported device (need sm_100)"}

# symbols include/hp.h declares (checked by tests/test_abi.py)
EXPORTS = ["hp_default_params", "hp_ctx_create", "hp_ctx_destroy", "hp_status_str",
           "hp_last_error", "hp_version", "hp_segment_tile", "hp_features_tile",
           "hp_process_tile", "hp_run_tiles", "hp_stage_run", "hp_set_stage_timing",
           "hp_get_stage_times", "hp_stage_times_accum", "hp_launch_count", "hp_reduce_rows",
           "hp_group_center", "hp_group_std", "hp_run_tiles_jpeg", "hp_process_tile_jpeg",
           "hp_decode_jpeg", "hp_jpeg_info"]


def jpeg_info(jpeg):
    """hp_jpeg_info (host only): {'width', 'height', 'sampling' (444 / 420), 'restart_interval'
    (MCUs, 0 = none), 'n_intervals'} of a JPEG file; raises HPError (status 5 = outside the
    decoder's scope, 1 = malformed)."""
    a = np.ascontiguousarray(np.frombuffer(bytes(jpeg), np.uint8) if isinstance(jpeg, (bytes, bytearray))
                             else jpeg, dtype=np.uint8)
    v = [C.c_int32() for _ in range(5)]
    st = lib().hp_jpeg_info(a.ctypes.data_as(C.c_void_p), a.nbytes, *[C.byref(x) for x in v])
    if st != 0:
        raise HPError(st, "hp_jpeg_info")
    return dict(zip(["width", "height", "sampling", "restart_interval", "n_intervals"], [x.value for x in v]))


class HPError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Params(C.Structure):
    _fields_ = [("q", (C.c_float * 3) * 3), ("g_scale", C.c_float), ("bg_rgb_min", C.c_int32),
                ("bg_skip_frac", C.c_float), ("rbc_t1", C.c_int32), ("rbc_t2", C.c_int32),
                ("open_diam", C.c_int32), ("g1", C.c_int32), ("cand_min_area", C.c_int32),
                ("cand_max_area", C.c_int32), ("h", C.c_float), ("obj_min_area", C.c_int32),
                ("obj_max_area", C.c_int32), ("glcm_levels", C.c_int32), ("canny_low", C.c_int32),
                ("canny_high", C.c_int32)]

    def to_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_ if f != "q"}
        d["q"] = [[self.q[k][j] for j in range(3)] for k in range(3)]
        return d

    @classmethod
    def from_dict(cls, d):
        p = cls()
        for f, _ in cls._fields_:
            if f == "q":
                for k in range(3):
                    for j in range(3):
                        p.q[k][j] = d["q"][k][j]
            else:
                setattr(p, f, d[f])
        return p


class Config(C.Structure):
    _fields_ = [("device", C.c_int32), ("max_width", C.c_int32), ("max_height", C.c_int32),
                ("n_slots", C.c_int32), ("max_objects", C.c_int32), ("params", Params)]


class Image(C.Structure):
    _fields_ = [("data", C.c_void_p), ("width", C.c_int32), ("height", C.c_int32),
                ("pitch_bytes", C.c_int64)]


class Labels(C.Structure):
    _fields_ = [("labels", C.c_void_p), ("labels_pitch_elems", C.c_int64),
                ("n_objects_dev", C.c_void_p)]


class FeatureTable(C.Structure):
    _fields_ = [("label", C.c_void_p), ("flags", C.c_void_p), ("feat", C.c_void_p),
                ("capacity", C.c_int32), ("n_rows_dev", C.c_void_p)]


class StageIO(C.Structure):
    _fields_ = [("in_", C.c_void_p * 4), ("out", C.c_void_p * 4), ("width", C.c_int32),
                ("height", C.c_int32)]


NEXT_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64),
                      C.POINTER(C.c_int64))
DONE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, C.c_int32, C.POINTER(C.c_int32),
                      C.POINTER(C.c_int32), C.POINTER(C.c_float), C.c_int)


class TileSource(C.Structure):
    _fields_ = [("next", NEXT_FN), ("user", C.c_void_p), ("width", C.c_int32),
                ("height", C.c_int32)]


class JpegSource(C.Structure):
    """hp_jpeg_source: next(user, &host_jpeg, &nbytes, &tile_id) -> 0 / 1 (drained)."""
    _fields_ = [("next", NEXT_FN), ("user", C.c_void_p), ("width", C.c_int32), ("height", C.c_int32)]


class RowArena(C.Structure):
    """hp_row_arena: device pointers (tile i64[cap], label i32[cap], flags i32[cap],
    feat f32[cap][36]), capacity, cursor (one device i64)."""
    _fields_ = [("tile", C.c_void_p), ("label", C.c_void_p), ("flags", C.c_void_p),
                ("feat", C.c_void_p), ("capacity", C.c_int64), ("cursor", C.c_void_p)]


class ResultSink(C.Structure):
    _fields_ = [("done", DONE_FN), ("user", C.c_void_p), ("arena", C.POINTER(RowArena))]


_lib = None


def lib():
    """Load libhp.so (built in-tree by paper_1209_3332_b200/build.py).  Raises if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(f"libhp.so not built ({SO_PATH}); run python -m "
                              "paper_1209_3332_b200.build or __graft_entry__.build()")
        L = C.CDLL(SO_PATH)
        P, i32 = C.c_void_p, C.c_int32
        sig = {
            "hp_default_params": (None, [C.POINTER(Params)]),
            "hp_ctx_create": (C.c_int, [C.POINTER(Config), C.POINTER(C.c_void_p)]),
            "hp_ctx_destroy": (C.c_int, [P]),
            "hp_status_str": (C.c_char_p, [C.c_int]),
            "hp_last_error": (C.c_char_p, [P]),
            "hp_version": (i32, []),
            "hp_segment_tile": (C.c_int, [P, i32, C.POINTER(Image), C.POINTER(Labels), P]),
            "hp_features_tile": (C.c_int, [P, i32, C.POINTER(Image), C.POINTER(Labels),
                                           C.POINTER(FeatureTable), P]),
            "hp_process_tile": (C.c_int, [P, i32, C.POINTER(Image), C.POINTER(Labels),
                                          C.POINTER(FeatureTable), P]),
            "hp_run_tiles": (C.c_int, [P, C.POINTER(TileSource), C.POINTER(ResultSink)]),
            "hp_stage_run": (C.c_int, [P, i32, C.c_int, C.POINTER(StageIO), P]),
            "hp_set_stage_timing": (C.c_int, [P, i32]),
            "hp_get_stage_times": (C.c_int, [P, i32, C.POINTER(C.c_float)]),
            "hp_stage_times_accum": (C.c_int, [P, C.POINTER(C.c_float), C.POINTER(C.c_int32)]),
            "hp_launch_count": (C.c_int64, []),
            "hp_reduce_rows": (C.c_int, [P, P, P, i32, P, P, P]),
            "hp_group_center": (C.c_int, [P, P, P, i32, P, P, P, P]),
            "hp_group_std": (C.c_int, [P, P, P, i32, P, P, P]),
            "hp_run_tiles_jpeg": (C.c_int, [P, C.POINTER(JpegSource), C.POINTER(ResultSink)]),
            "hp_process_tile_jpeg": (C.c_int, [P, i32, P, C.c_int64, C.POINTER(Labels), C.POINTER(FeatureTable),
                                               P, P]),
            "hp_decode_jpeg": (C.c_int, [P, i32, P, C.c_int64, P, C.c_int64, P]),
            "hp_jpeg_info": (C.c_int, [P, C.c_int64, P, P, P, P, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def launch_count() -> int:
    """libhp kernel launches issued by this process so far."""
    return int(lib().hp_launch_count())


def default_params() -> Params:
    p = Params()
    lib().hp_default_params(C.byref(p))
    return p


def _ptr(t):
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


class Context:
    """One hp_ctx: scratch for n_slots tiles of up to max_width x max_height on `device`."""

    def __init__(self, device=0, max_width=4096, max_height=4096, n_slots=1, max_objects=65536,
                 params: Params | None = None):
        cfg = Config(device, max_width, max_height, n_slots, max_objects,
                     params if params is not None else default_params())
        h = C.c_void_p()
        st = lib().hp_ctx_create(C.byref(cfg), C.byref(h))
        if st != 0:
            raise HPError(st, "hp_ctx_create")
        self._h = h
        self.cfg = cfg

    def close(self):
        if getattr(self, "_h", None):
            lib().hp_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _chk(self, st, what):
        if st != 0:
            msg = lib().hp_last_error(self._h)
            raise HPError(st, f"{what}: {msg.decode() if msg else ''}")

    @staticmethod
    def image(rgb):
        """rgb: uint8 tensor [H, W, 3] (device for tile calls)."""
        h, w = rgb.shape[0], rgb.shape[1]
        return Image(rgb.data_ptr(), w, h, rgb.stride(0) * rgb.element_size())

    def segment_tile(self, slot, rgb, labels, n_objects, stream=None):
        im = self.image(rgb)
        lab = Labels(labels.data_ptr(), labels.stride(0), n_objects.data_ptr())
        self._chk(lib().hp_segment_tile(self._h, slot, C.byref(im), C.byref(lab), _stream(stream)),
                  "hp_segment_tile")

    def features_tile(self, slot, rgb, labels, n_objects, t_label, t_flags, t_feat, n_rows,
                      stream=None):
        im = self.image(rgb)
        lab = Labels(labels.data_ptr(), labels.stride(0), n_objects.data_ptr())
        tab = FeatureTable(t_label.data_ptr(), t_flags.data_ptr(), t_feat.data_ptr(),
                           t_label.shape[0], n_rows.data_ptr())
        self._chk(lib().hp_features_tile(self._h, slot, C.byref(im), C.byref(lab), C.byref(tab),
                                         _stream(stream)), "hp_features_tile")

    def reduce_rows(self, feat, off, out, out_count, stream=None):
        """hp_reduce_rows: per group g, sums and sums of squares (f64) of the feature rows
        [off[g], off[g+1]) of feat ([n, 36] f32); all device tensors."""
        self._chk(lib().hp_reduce_rows(self._h, feat.data_ptr(), off.data_ptr(), off.shape[0] - 1,
                                       out.data_ptr(), out_count.data_ptr(), _stream(stream)), "hp_reduce_rows")

    def group_center(self, feat, off, sums, count, mean_m2, stream=None):
        """hp_group_center: per group, mean = sums[..., 0] / count and the sum over these rows
        of (x - mean)^2 -> mean_m2 [G, 36, 2] f64 (all device tensors; sums/count are totals)."""
        self._chk(lib().hp_group_center(self._h, feat.data_ptr(), off.data_ptr(), off.shape[0] - 1,
                                        sums.data_ptr(), count.data_ptr(), mean_m2.data_ptr(), _stream(stream)),
                  "hp_group_center")

    def group_std(self, mean_m2, count, mean, std, stream=None):
        """hp_group_std: mean [G, 36] and population std = sqrt(m2 / count) [G, 36] (f64)."""
        self._chk(lib().hp_group_std(self._h, mean_m2.data_ptr(), count.data_ptr(), count.shape[0],
                                     mean.data_ptr(), std.data_ptr(), _stream(stream)), "hp_group_std")

    def process_tile(self, slot, rgb, labels, n_objects, t_label, t_flags, t_feat, n_rows,
                     stream=None):
        im = self.image(rgb)
        lab = Labels(labels.data_ptr(), labels.stride(0), n_objects.data_ptr())
        tab = FeatureTable(t_label.data_ptr(), t_flags.data_ptr(), t_feat.data_ptr(),
                           t_label.shape[0], n_rows.data_ptr())
        self._chk(lib().hp_process_tile(self._h, slot, C.byref(im), C.byref(lab), C.byref(tab),
                                        _stream(stream)), "hp_process_tile")

    def stage_run(self, slot, stage, ins, outs, width, height, stream=None):
        io = StageIO()
        for k, t in enumerate(ins):
            io.in_[k] = None if t is None else t.data_ptr()
        for k, t in enumerate(outs):
            io.out[k] = None if t is None else t.data_ptr()
        io.width, io.height = width, height
        st = STAGE[stage] if isinstance(stage, str) else stage
        self._chk(lib().hp_stage_run(self._h, slot, st, C.byref(io), _stream(stream)),
                  f"hp_stage_run({stage})")

    def set_stage_timing(self, on=True):
        self._chk(lib().hp_set_stage_timing(self._h, 1 if on else 0), "hp_set_stage_timing")

    def stage_times(self, slot=0):
        ms = (C.c_float * 11)()
        self._chk(lib().hp_get_stage_times(self._h, slot, ms), "hp_get_stage_times")
        return list(ms)

    def stage_times_accum(self):
        """(sum of S1..S11 ms over the recorded tiles, number of tiles)."""
        ms = (C.c_float * 11)()
        n = C.c_int32()
        self._chk(lib().hp_stage_times_accum(self._h, ms, C.byref(n)), "hp_stage_times_accum")
        return list(ms), int(n.value)

    def run_tiles(self, next_tile, on_done, width, height, arena=None):
        """Demand-driven driver.  next_tile() -> (host_ptr:int, pitch:int, tile_id:int) or
        None when drained; host memory must be pinned and stay valid until on_done for that
        tile.  on_done(tile_id, label[n], flags[n], feat[n, 36], status) gets numpy COPIES.
        With arena = (tile_ptr, label_ptr, flags_ptr, feat_ptr, capacity, cursor_ptr) (device
        pointers, hp_row_arena) the rows are appended on the device instead and
        on_done(tile_id, n_rows, status) is called."""
        self._run(lib().hp_run_tiles, TileSource, "hp_run_tiles", next_tile, on_done, width, height, arena)

    def run_tiles_jpeg(self, next_tile, on_done, width, height, arena=None):
        """hp_run_tiles_jpeg (NEXT-3 compressed ingest): as run_tiles, but next_tile() returns
        (host_ptr, nbytes, tile_id) of a baseline JPEG file of a width x height tile (pinned
        memory recommended).  A file the decoder rejects is delivered with a nonzero status
        and no rows."""
        self._run(lib().hp_run_tiles_jpeg, JpegSource, "hp_run_tiles_jpeg", next_tile, on_done, width, height,
                  arena)

    def _run(self, fn, src_type, name, next_tile, on_done, width, height, arena):
        # ctypes prints and swallows an exception raised inside a C callback, so both
        # callbacks store the first one; after it no further tile is fed, and it is re-raised
        # once the driver has returned (the tiles already in flight are drained by then).
        keep = []
        err = []

        def _next(user, pp, ppitch, ptid):
            if err:
                return 1
            try:
                r = next_tile()
            except BaseException as e:  # noqa: BLE001 -- never raise through C
                err.append(e)
                return 1
            if r is None:
                return 1
            ptr, pitch, tid = r
            pp[0] = ptr
            ppitch[0] = pitch
            ptid[0] = tid
            return 0

        def _done(user, tid, n, plab, pflags, pfeat, st):
            if err:
                return
            try:
                if arena is not None:
                    on_done(int(tid), int(n), int(st))
                    return
                lab = np.ctypeslib.as_array(plab, shape=(max(n, 1),))[:n].copy()
                fl = np.ctypeslib.as_array(pflags, shape=(max(n, 1),))[:n].copy()
                ft = np.ctypeslib.as_array(pfeat, shape=(max(n, 1) * NFEAT,))[:n * NFEAT].copy()
                on_done(int(tid), lab, fl, ft.reshape(n, NFEAT), int(st))
            except BaseException as e:  # noqa: BLE001
                err.append(e)

        nf, df = NEXT_FN(_next), DONE_FN(_done)
        keep += [nf, df]
        src = src_type(nf, None, width, height)
        ar = None if arena is None else RowArena(*arena)
        sink = ResultSink(df, None, C.pointer(ar) if ar is not None else None)
        keep.append(ar)
        st = fn(self._h, C.byref(src), C.byref(sink))
        if err:
            raise err[0]
        self._chk(st, name)

    @staticmethod
    def _host_buf(jpeg):
        """(pointer, nbytes, owner) of a host JPEG buffer: a numpy u8 array or a (pinned) CPU
        tensor; the caller keeps `owner` alive across the call (a contiguous copy of a strided
        array lives only there)."""
        if hasattr(jpeg, "data_ptr"):
            if not jpeg.is_contiguous():
                jpeg = jpeg.contiguous()
            return jpeg.data_ptr(), jpeg.numel() * jpeg.element_size(), jpeg
        a = np.ascontiguousarray(jpeg, dtype=np.uint8)
        return a.ctypes.data, a.nbytes, a

    def process_tile_jpeg(self, slot, jpeg, labels, n_objects, t_label, t_flags, t_feat, n_rows,
                          decode_err=None, stream=None):
        """hp_process_tile_jpeg: one JPEG tile (host bytes, kept alive until the stream is
        done) through both stages; decode_err: optional device int32 tensor."""
        ptr, nb, _owner = self._host_buf(jpeg)
        lab = Labels(labels.data_ptr(), labels.stride(0), n_objects.data_ptr())
        tab = FeatureTable(t_label.data_ptr(), t_flags.data_ptr(), t_feat.data_ptr(),
                           t_label.shape[0], n_rows.data_ptr())
        self._chk(lib().hp_process_tile_jpeg(self._h, slot, C.c_void_p(ptr), nb, C.byref(lab), C.byref(tab),
                                             None if decode_err is None else C.c_void_p(decode_err.data_ptr()),
                                             _stream(stream)), "hp_process_tile_jpeg")

    def decode_jpeg(self, slot, jpeg, rgb_out, stream=None):
        """hp_decode_jpeg: decoded RGB into the device tensor rgb_out [H, W, 3] (synchronises)."""
        ptr, nb, _owner = self._host_buf(jpeg)
        self._chk(lib().hp_decode_jpeg(self._h, slot, C.c_void_p(ptr), nb, C.c_void_p(rgb_out.data_ptr()),
                                       rgb_out.stride(0) * rgb_out.element_size(), _stream(stream)),
                  "hp_decode_jpeg")
