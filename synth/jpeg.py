"""Seeded JPEG encoding of synthetic tiles for the compressed-ingest path (SURVEY.md §8(f)
NEXT-3; tile I/O is the bottleneck).  Input preparation only: the bytes
come from OpenCV's encoder (libjpeg), baseline sequential Huffman, 4:4:4, with a restart
interval so the decoder can run one restart interval per thread.  No decoding arithmetic
lives here (the oracle and libhp each decode independently)."""
from __future__ import annotations

import numpy as np

DEFAULT_QUALITY = 90
DEFAULT_RST = 4  # MCUs per restart interval


def encode_tile(rgb: np.ndarray, quality: int = DEFAULT_QUALITY, rst: int = DEFAULT_RST,
                sampling: str = "444", progressive: bool = False) -> np.ndarray:
    """RGB u8 [H, W, 3] -> JPEG bytes (u8 array)."""
    import cv2
    bgr = np.ascontiguousarray(np.asarray(rgb, np.uint8)[:, :, ::-1])
    params = [cv2.IMWRITE_JPEG_QUALITY, int(quality), cv2.IMWRITE_JPEG_RST_INTERVAL, int(rst),
              cv2.IMWRITE_JPEG_SAMPLING_FACTOR, getattr(cv2, f"IMWRITE_JPEG_SAMPLING_FACTOR_{sampling}")]
    if progressive:
        params += [cv2.IMWRITE_JPEG_PROGRESSIVE, 1]
    ok, buf = cv2.imencode(".jpg", bgr, params)
    if not ok:
        raise RuntimeError("cv2.imencode failed")
    return np.ascontiguousarray(buf.reshape(-1), np.uint8)
