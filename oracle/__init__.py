"""ctypes binding of liboracle -- the plain CPU oracle of the per-tile pipeline.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  The product path
(paper_1209_3332_b200, libhp) never imports it and shares no code with it.

Every wrapper takes/returns numpy arrays and calls the C function of the same name
(oracle/oracle.h), which cites the passage of PAPER.md / SURVEY.md §8(c) it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")

NFEAT = 36
FLAG_RBC_HI, FLAG_RBC_LO, FLAG_R_GT_B, FLAG_BG = 1, 2, 4, 8
OBJ_TOUCHES_BORDER = 1


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (-O2, no FMA contraction, no fast-math)."""
    srcs = [_SRC, os.path.join(_HERE, "jpeg.cpp")]
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            [os.path.getmtime(f) for f in srcs] + [os.path.getmtime(os.path.join(_HERE, "oracle.h"))]):
        cmd = ["g++", "-O2", "-ffp-contract=off", "-fno-fast-math", "-ftree-vectorize", "-std=c++17", "-fPIC",
               "-shared", "-o", _SO] + srcs
        subprocess.check_call(cmd, cwd=_HERE)
    return _SO


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


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        i32, i64 = C.c_int32, C.c_int64
        sig = {
            "or_default_params": (None, [C.POINTER(Params)]),
            "or_cd": (C.c_int, [P, C.c_int, C.c_int, i64, C.POINTER(Params), P, P, P]),
            "or_rbc": (C.c_int, [P, C.c_int, C.c_int, P]),
            "or_open": (C.c_int, [P, C.c_int, C.c_int, C.c_int, P]),
            "or_erode": (C.c_int, [P, C.c_int, C.c_int, C.c_int, P]),
            "or_dilate": (C.c_int, [P, C.c_int, C.c_int, C.c_int, P]),
            "or_recon_u8": (C.c_int, [P, P, C.c_int, C.c_int, P, P]),
            "or_recon_f32": (C.c_int, [P, P, P, C.c_int, C.c_int, P]),
            "or_recon_to_nuclei": (C.c_int, [P, P, P, C.c_int, C.c_int, C.c_int, P, P]),
            "or_ccl": (C.c_int, [P, C.c_int, C.c_int, C.c_int, P, P]),
            "or_area_threshold": (C.c_int, [P, C.c_int, C.c_int, C.c_int, C.c_int, P]),
            "or_fill_holes": (C.c_int, [P, C.c_int, C.c_int, P]),
            "or_edt": (C.c_int, [P, C.c_int, C.c_int, P, P]),
            "or_markers": (C.c_int, [P, P, C.c_int, C.c_int, C.c_float, P, P, P]),
            "or_watershed": (C.c_int, [P, P, P, C.c_int, C.c_int, P, P, P, P]),
            "or_bwlabel": (C.c_int, [P, C.c_int, C.c_int, C.c_int, C.c_int, P, P]),
            "or_features": (C.c_int, [P, P, C.c_int, C.c_int, C.c_int, i32, P, P, P, P]),
            "or_segment_tile": (C.c_int, [P, C.c_int, C.c_int, i64, C.POINTER(Params), P, P, P]),
            "or_process_tile": (C.c_int, [P, C.c_int, C.c_int, i64, C.POINTER(Params), P, i32,
                                          P, P, P, P, P]),
            "or_aggregate": (C.c_int, [P, C.c_int, P, C.c_int, P, P, P]),
            "or_jpeg_decode": (C.c_int, [P, i64, P, P, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def _chk(rc, name):
    if rc != 0:
        raise RuntimeError(f"{name} returned {rc}")


def default_params() -> Params:
    p = Params()
    lib().or_default_params(C.byref(p))
    return p


def cd(rgb, params=None):
    rgb = _u8(rgb)
    h, w = rgb.shape[:2]
    params = params or default_params()
    g = np.empty((h, w), np.uint8)
    fl = np.empty((h, w), np.uint8)
    nbg = np.zeros(1, np.int64)
    _chk(lib().or_cd(_p(rgb), w, h, 3 * w, C.byref(params), _p(g), _p(fl), _p(nbg)), "or_cd")
    return g, fl, int(nbg[0])


def rbc(flags):
    flags = _u8(flags)
    h, w = flags.shape
    out = np.empty((h, w), np.uint8)
    _chk(lib().or_rbc(_p(flags), w, h, _p(out)), "or_rbc")
    return out


def _morph(name, g, diam):
    g = _u8(g)
    h, w = g.shape
    out = np.empty((h, w), np.uint8)
    _chk(getattr(lib(), name)(_p(g), w, h, diam, _p(out)), name)
    return out


def erode(g, diam=19):
    return _morph("or_erode", g, diam)


def dilate(g, diam=19):
    return _morph("or_dilate", g, diam)


def open_(g, diam=19):
    return _morph("or_open", g, diam)


def recon_u8(marker, mask, with_stats=False):
    marker, mask = _u8(marker), _u8(mask)
    h, w = mask.shape
    out = np.empty((h, w), np.uint8)
    st = np.zeros(2, np.int64)
    _chk(lib().or_recon_u8(_p(marker), _p(mask), w, h, _p(out), _p(st)), "or_recon_u8")
    return (out, st) if with_stats else out


def recon_f32(marker, mask, dom=None):
    marker = np.ascontiguousarray(marker, np.float32)
    mask = np.ascontiguousarray(mask, np.float32)
    h, w = mask.shape
    out = np.empty((h, w), np.float32)
    d = None if dom is None else _u8(dom)
    _chk(lib().or_recon_f32(_p(marker), _p(mask), _p(d), w, h, _p(out)), "or_recon_f32")
    return out


def recon_to_nuclei(g, open_img, rbc_img, g1=50, with_recon=False):
    g, open_img, rbc_img = _u8(g), _u8(open_img), _u8(rbc_img)
    h, w = g.shape
    cand = np.empty((h, w), np.uint8)
    rec = np.empty((h, w), np.uint8)
    _chk(lib().or_recon_to_nuclei(_p(g), _p(open_img), _p(rbc_img), w, h, g1, _p(cand), _p(rec)),
         "or_recon_to_nuclei")
    return (cand, rec) if with_recon else cand


def ccl(fg, conn=8):
    fg = _u8(fg)
    h, w = fg.shape
    lab = np.empty((h, w), np.int32)
    n = np.zeros(1, np.int32)
    _chk(lib().or_ccl(_p(fg), w, h, conn, _p(lab), _p(n)), "or_ccl")
    return lab, int(n[0])


def area_threshold(cand, amin=11, amax=1000):
    cand = _u8(cand)
    h, w = cand.shape
    out = np.empty((h, w), np.uint8)
    _chk(lib().or_area_threshold(_p(cand), w, h, amin, amax, _p(out)), "or_area_threshold")
    return out


def fill_holes(big0):
    big0 = _u8(big0)
    h, w = big0.shape
    out = np.empty((h, w), np.uint8)
    _chk(lib().or_fill_holes(_p(big0), w, h, _p(out)), "or_fill_holes")
    return out


def edt(F):
    F = _u8(F)
    h, w = F.shape
    d2 = np.empty((h, w), np.uint32)
    dist = np.empty((h, w), np.float32)
    _chk(lib().or_edt(_p(F), w, h, _p(d2), _p(dist)), "or_edt")
    return d2, dist


def markers(dist, F, hh=1.0):
    dist = np.ascontiguousarray(dist, np.float32)
    F = _u8(F)
    h, w = F.shape
    ML = np.empty((h, w), np.int32)
    J = np.empty((h, w), np.float32)
    n = np.zeros(1, np.int32)
    _chk(lib().or_markers(_p(dist), _p(F), w, h, hh, _p(ML), _p(J), _p(n)), "or_markers")
    return ML, J, int(n[0])


def watershed(dist, ML, F):
    dist = np.ascontiguousarray(dist, np.float32)
    ML = np.ascontiguousarray(ML, np.int32)
    F = _u8(F)
    h, w = F.shape
    c = np.empty((h, w), np.float32)
    d = np.empty((h, w), np.int32)
    L = np.empty((h, w), np.int32)
    split = np.empty((h, w), np.uint8)
    _chk(lib().or_watershed(_p(dist), _p(ML), _p(F), w, h, _p(c), _p(d), _p(L), _p(split)),
         "or_watershed")
    return split, c, d, L


def bwlabel(split, amin=21, amax=1000):
    split = _u8(split)
    h, w = split.shape
    lab = np.empty((h, w), np.int32)
    n = np.zeros(1, np.int32)
    _chk(lib().or_bwlabel(_p(split), w, h, amin, amax, _p(lab), _p(n)), "or_bwlabel")
    return lab, int(n[0])


def canny(g, low=100, high=200):
    """Feature-stage Canny edges (0/1) of g: cv2.Canny(g, low, high) written out (C22)."""
    g = _u8(g)
    h, w = g.shape
    out = np.empty((h, w), np.uint8)
    _chk(lib().or_canny(_p(g), w, h, int(low), int(high), _p(out)), "or_canny")
    return out


def features(labels, g, cap=None, canny_low=100, canny_high=200):
    labels = np.ascontiguousarray(labels, np.int32)
    g = _u8(g)
    h, w = g.shape
    if cap is None:
        cap = max(1, int(len(np.unique(labels))))
    rl = np.zeros(cap, np.int32)
    rf = np.zeros(cap, np.int32)
    ft = np.zeros((cap, NFEAT), np.float32)
    n = np.zeros(1, np.int32)
    _chk(lib().or_features(_p(labels), _p(g), w, h, 8, int(canny_low), int(canny_high), cap, _p(rl), _p(rf),
                           _p(ft), _p(n)), "or_features")
    k = int(n[0])
    return rl[:k], rf[:k], ft[:k]


def segment_tile(rgb, params=None, with_times=False):
    rgb = _u8(rgb)
    h, w = rgb.shape[:2]
    params = params or default_params()
    lab = np.empty((h, w), np.int32)
    n = np.zeros(1, np.int32)
    t = np.zeros(11, np.float64)
    _chk(lib().or_segment_tile(_p(rgb), w, h, 3 * w, C.byref(params), _p(lab), _p(n), _p(t)),
         "or_segment_tile")
    return (lab, int(n[0]), t) if with_times else (lab, int(n[0]))


def process_tile(rgb, params=None, cap=65536, with_times=False):
    """The whole hot path (S1..S11) for one tile: labels + feature rows."""
    rgb = _u8(rgb)
    h, w = rgb.shape[:2]
    params = params or default_params()
    lab = np.empty((h, w), np.int32)
    rl = np.zeros(cap, np.int32)
    rf = np.zeros(cap, np.int32)
    ft = np.zeros((cap, NFEAT), np.float32)
    n = np.zeros(1, np.int32)
    t = np.zeros(11, np.float64)
    _chk(lib().or_process_tile(_p(rgb), w, h, 3 * w, C.byref(params), _p(lab), cap, _p(rl),
                               _p(rf), _p(ft), _p(n), _p(t)), "or_process_tile")
    k = int(n[0])
    out = (lab, rl[:k], rf[:k], ft[:k])
    return out + (t,) if with_times else out


def aggregate(feat, off):
    """NEXT-4: per group g = rows [off[g], off[g+1]) of feat [n, F] f32 ->
    (count [G] int64, mean [G, F] f64, population std [G, F] f64), NaN for an empty group."""
    feat = np.ascontiguousarray(feat, dtype=np.float32)
    if feat.ndim == 1:
        feat = feat.reshape(-1, 1)
    off = np.ascontiguousarray(off, dtype=np.int64)
    G, F = len(off) - 1, feat.shape[1]
    cnt = np.empty(G, np.int64)
    mean = np.empty((G, F), np.float64)
    std = np.empty((G, F), np.float64)
    fp = feat if feat.size else np.zeros((1, F), np.float32)
    _chk(lib().or_aggregate(_p(fp), F, _p(off), G, _p(cnt), _p(mean), _p(std)), "or_aggregate")
    return cnt, mean, std


def jpeg_decode(data):
    """NEXT-3: baseline JPEG bytes -> RGB u8 [H, W, 3] (T.81 decoding,
    readings J1-J2: IJG islow IDCT, JFIF colour).  Raises on unsupported / invalid input."""
    buf = np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else \
        np.ascontiguousarray(data, np.uint8)
    w = np.zeros(1, np.int32)
    h = np.zeros(1, np.int32)
    _chk(lib().or_jpeg_decode(_p(buf), buf.size, _p(w), _p(h), None), "or_jpeg_decode (header)")
    out = np.empty((int(h[0]), int(w[0]), 3), np.uint8)
    _chk(lib().or_jpeg_decode(_p(buf), buf.size, _p(w), _p(h), _p(out)), "or_jpeg_decode")
    return out
