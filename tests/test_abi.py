"""CPU-side checks of the boundary (no GPU needed): libhp.so loads, exports every symbol
include/hp.h declares, its defaults agree with the oracle's independently computed ones,
hp_ctx_create refuses to run without a B200 (no CPU fallback), and the product package
never imports the oracle."""
import ctypes as C
import os
import re

import pytest

import oracle
import paper_1209_3332_b200 as P
from paper_1209_3332_b200 import hp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "hp.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hp_[a-z_0-9]+)\s*\(", txt)) - {"hp_stream"})


def test_exports_match_header():
    L = hp.lib()
    decl = _declared()
    assert set(decl) == set(hp.EXPORTS), decl
    for name in decl:
        assert hasattr(L, name), name
    assert L.hp_version() == 2


def test_default_params_agree_with_oracle():
    a = P.default_params().to_dict()
    b = oracle.default_params().to_dict()
    assert a == b


def test_struct_layouts():
    assert C.sizeof(hp.Params) == 9 * 4 + 15 * 4  # q[3][3] + 15 scalar fields
    # the C side writes exactly sizeof(hp_params) bytes: ..., glcm_levels, canny_low, canny_high
    buf = (C.c_uint8 * 200)(*([0xAB] * 200))
    hp.lib().hp_default_params(C.cast(buf, C.POINTER(hp.Params)))
    assert all(b == 0xAB for b in buf[96:])
    assert int.from_bytes(bytes(buf[84:88]), "little") == 8
    assert int.from_bytes(bytes(buf[88:92]), "little") == 100 and int.from_bytes(bytes(buf[92:96]), "little") == 200
    assert C.sizeof(hp.Config) == 5 * 4 + C.sizeof(hp.Params)
    assert C.sizeof(hp.Image) == 24 and C.sizeof(hp.Labels) == 24
    assert C.sizeof(hp.StageIO) == 72


def test_status_strings():
    L = hp.lib()
    assert L.hp_status_str(0) == b"ok"
    assert L.hp_status_str(5).startswith(b"unsupported")


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(hp.HPError) as e:
        hp.Context(0, 64, 64, 1, 16)
    assert e.value.status == 5


def test_invalid_config_rejected():
    cfg = hp.Config(0, 0, 64, 1, 16, P.default_params())
    h = C.c_void_p()
    assert hp.lib().hp_ctx_create(C.byref(cfg), C.byref(h)) == 1
    p = P.default_params()
    p.open_diam = 18
    cfg = hp.Config(0, 64, 64, 1, 16, p)
    assert hp.lib().hp_ctx_create(C.byref(cfg), C.byref(h)) == 1
    for lo, hi in [(-1, 10), (200, 100)]:          # reading C22: 0 <= canny_low <= canny_high
        p = P.default_params()
        p.canny_low, p.canny_high = lo, hi
        cfg = hp.Config(0, 64, 64, 1, 16, p)
        assert hp.lib().hp_ctx_create(C.byref(cfg), C.byref(h)) == 1


def test_product_does_not_touch_oracle():
    pkg = os.path.join(ROOT, "paper_1209_3332_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "oracle.h" not in src and "liboracle" not in src, f


def test_struct_layouts_match_header(tmp_path):
    """Every ctypes structure of the binding has the size and field offsets the C compiler
    gives the same struct from include/hp.h (compiled here with gcc)."""
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    pairs = [("hp_params", hp.Params), ("hp_config", hp.Config), ("hp_image", hp.Image),
             ("hp_labels", hp.Labels), ("hp_feature_table", hp.FeatureTable),
             ("hp_stage_io", hp.StageIO), ("hp_tile_source", hp.TileSource),
             ("hp_row_arena", hp.RowArena), ("hp_result_sink", hp.ResultSink),
             ("hp_jpeg_source", hp.JpegSource)]
    cname = {"in_": "in"}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "hp.h"', "int main(void) {"]
    expect = []
    for cs, py in pairs:
        lines.append(f'printf("%zu\\n", sizeof({cs}));')
        expect.append(C.sizeof(py))
        for f, _ in py._fields_:
            lines.append(f'printf("%zu\\n", offsetof({cs}, {cname.get(f, f)}));')
            expect.append(getattr(py, f).offset)
    lines += ["return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run([cc, "-std=c99", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert got == expect


def test_feature_names_follow_header_enum():
    """hp.FEATURE_NAMES has one name per HP_F_* column, in the enum's order."""
    txt = open(os.path.join(ROOT, "include", "hp.h")).read()
    body = txt[txt.index("HP_F_AREA = 0"):txt.index("HP_NFEAT = 36")]
    enum = re.findall(r"\bHP_F_([A-Z_0-9]+)", body)
    assert len(enum) == hp.NFEAT == len(hp.FEATURE_NAMES)
    for e, n in zip(enum, hp.FEATURE_NAMES):
        assert e.lower() == n, (e, n)
