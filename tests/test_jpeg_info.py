"""Host-side JPEG header parsing of libhp (hp_jpeg_info; CPU only): frame size, sampling and
restart layout agree with the encoder's parameters and OpenCV's decode, and files outside the
GPU decoder's scope (reading J3) are refused with the status the JPEG calls return."""
import cv2
import numpy as np
import pytest

from paper_1209_3332_b200 import hp
from synth.hne import TileSpec, make_tile
from synth.jpeg import encode_tile


@pytest.mark.parametrize("shape,rst,sampling", [((64, 64), 4, "444"), ((37, 53), 1, "444"), ((300, 257), 0, "444"),
                                                ((129, 200), 17, "420"), ((1, 300), 2, "420"), ((4096, 16), 64, "420")])
def test_header_fields(shape, rst, sampling):
    rgb = make_tile(sum(shape), TileSpec(*shape))["rgb"]
    buf = encode_tile(rgb, 85, rst, sampling=sampling)
    info = hp.jpeg_info(buf)
    h, w = cv2.imdecode(buf, cv2.IMREAD_COLOR).shape[:2]
    assert (info["width"], info["height"]) == (w, h) == (shape[1], shape[0])
    assert info["sampling"] == int(sampling)
    mcu = 8 if sampling == "444" else 16
    nmcu = -(-shape[0] // mcu) * -(-shape[1] // mcu)
    if rst == 0 or rst >= nmcu:
        assert info["restart_interval"] == 0 and info["n_intervals"] == 1
    else:
        assert info["restart_interval"] == rst and info["n_intervals"] == -(-nmcu // rst)


def test_refusals():
    rgb = make_tile(9, TileSpec(48, 48))["rgb"]
    with pytest.raises(hp.HPError) as e:
        hp.jpeg_info(encode_tile(rgb, 90, 2, sampling="422"))
    assert e.value.status == 5
    with pytest.raises(hp.HPError) as e:
        hp.jpeg_info(encode_tile(rgb, 90, 0, progressive=True))
    assert e.value.status == 5
    grey = cv2.imencode(".jpg", rgb[:, :, 0])[1].reshape(-1)
    with pytest.raises(hp.HPError) as e:
        hp.jpeg_info(grey)
    assert e.value.status == 5
    good = encode_tile(rgb, 90, 2)
    for bad in (good[:40], np.zeros(16, np.uint8), good[2:]):
        with pytest.raises(hp.HPError) as e:
            hp.jpeg_info(bad)
        assert e.value.status == 1
