"""CPU: IDX data files (dataset.hpp:84-196) through the C-ABI -- the reference's own
test_dataset.cpp cases (constructed fixture, malformed streams, gzip), plus a random
payload round trip."""
import gzip
import os
import struct

import numpy as np
import pytest


def be32(v):
    return struct.pack(">I", v)


def tiny_images():  # two 1x1 images with pixels {0, 255}
    return be32(0x803) + be32(2) + be32(1) + be32(1) + bytes([0, 255])


def tiny_labels():  # labels {1, 0}
    return be32(0x801) + be32(2) + bytes([1, 0])


def test_parse_idx_fixture(product):  # test_dataset.cpp:53-61
    X, y, nc = product.parse_idx(tiny_images(), tiny_labels())
    assert X.shape == (2, 1) and X[0, 0] == 0.0 and X[1, 0] == 1.0
    assert list(y) == [1, 0] and nc == 2


def test_parse_idx_rejects_malformed(product):  # test_dataset.cpp:63-81
    with pytest.raises(ValueError, match="magic"):
        product.parse_idx(tiny_labels(), tiny_labels())
    with pytest.raises(ValueError, match="magic"):
        product.parse_idx(tiny_images(), tiny_images())
    with pytest.raises(ValueError, match="payload"):
        product.parse_idx(tiny_images()[:-1], tiny_labels())
    extra = bytearray(tiny_labels())
    extra[7] = 3  # claims 3 labels
    with pytest.raises(ValueError):
        product.parse_idx(tiny_images(), bytes(extra))
    with pytest.raises(ValueError, match="offset"):
        product.parse_idx(bytes([0, 0]), tiny_labels())


def test_random_payload_and_gzip_files(product, tmp_path):  # test_dataset.cpp:92-131
    rng = np.random.default_rng(91)
    px = rng.integers(0, 256, size=5 * 3 * 2).astype(np.uint8)
    lab = rng.integers(0, 10, size=5).astype(np.uint8)
    img = be32(0x803) + be32(5) + be32(3) + be32(2) + px.tobytes()
    lb = be32(0x801) + be32(5) + lab.tobytes()
    X, y, nc = product.parse_idx(img, lb)
    assert np.array_equal(X, (px.astype(np.float64) / 255.0).astype(np.float32).reshape(5, 6))
    assert np.array_equal(y, lab.astype(np.int32)) and nc == int(lab.max()) + 1
    # serialize back (the reference's serialize_idx: round(x * 255))
    assert bytes(np.rint(X.astype(np.float64) * 255.0).astype(np.uint8).tobytes()) == px.tobytes()
    ip, lp = os.path.join(tmp_path, "img.idx.gz"), os.path.join(tmp_path, "lab.idx.gz")
    with gzip.open(ip, "wb") as f:
        f.write(img)
    with gzip.open(lp, "wb") as f:
        f.write(lb)
    X2, y2, _ = product.load_idx(ip, lp)
    assert np.array_equal(X2, X) and np.array_equal(y2, y)
    raw = os.path.join(tmp_path, "img.idx")
    with open(raw, "wb") as f:
        f.write(img)
    X3, _, _ = product.load_idx(raw, lp)  # mixed raw + gzip
    assert np.array_equal(X3, X)
    with pytest.raises(ValueError, match="cannot open"):
        product.load_idx(os.path.join(tmp_path, "missing-file.idx"), lp)
