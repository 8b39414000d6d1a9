"""Pin the CPU oracle (oracle/salr_oracle.py) against the reference's own
known-answer tests and the golden fixtures produced by running the real
reference (tests/golden/make_golden.py).  Nothing else may trust the oracle
before these pass."""

import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import salr_oracle as O


class TestKnownAnswers:
    """Reference KATs (pkg/tests/test_bitmap.py, test_acceptance.py)."""

    def test_popcount_exhaustive(self):  # test_bitmap.py:50-52
        for m in range(256):
            assert O.popcount8(m) == bin(m).count("1")

    def test_lut_exhaustive(self):  # test_bitmap.py:64-75, test_acceptance.py:328-337
        lut = O.build_lut()
        assert lut.shape == (256, 8) and lut.dtype == np.int8
        for m in range(256):
            seen = 0
            for t in range(8):
                if m >> t & 1:
                    assert lut[m, t] == seen
                    seen += 1
                else:
                    assert lut[m, t] == -1
        np.testing.assert_array_equal(lut[5], [0, -1, 1, -1, -1, -1, -1, -1])

    def test_byte_146(self):  # test_bitmap.py:84-89
        s = O.encode(np.array([[0.0, 1.5, 0.0, 0.0, -2.0, 0.0, 0.0, 3.0]]))
        assert s.bitmap.tolist() == [[146]]
        np.testing.assert_array_equal(s.values, np.float32([1.5, -2.0, 3.0]))

    def test_padding_and_signed_zero(self):  # test_bitmap.py:97-115
        assert np.all(O.encode(np.ones((3, 5))).bitmap == 0b00011111)
        s = O.encode(np.array([[-0.0, 1.0]]))
        assert s.nnz == 1 and s.bitmap.tolist() == [[2]]
        s = O.encode(np.array([[1e-60, 1.0]]))
        assert s.nnz == 1 and O.decode(s)[0, 0] == 0.0

    def test_compression_ratio(self):  # test_bitmap.py:372-382
        assert O.compression_ratio(4096, 4096, 0.5, 2, 0) == pytest.approx(1.7778, abs=1e-3)
        assert O.compression_ratio(4096, 4096, 0.9, 2, 0) == pytest.approx(6.1538, abs=1e-3)

    def test_kept_count(self):
        assert O.kept_count(0.5, 4096 * 4096) == 4096 * 4096 // 2
        assert O.kept_count(0.7, 100 * 100) == 3000


def _load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def test_codec_matches_reference_goldens():
    z = _load("codec.npz")
    for i in range(int(z["n"])):
        w = z[f"w_{i}"]
        s = O.encode(w)
        np.testing.assert_array_equal(s.bitmap, z[f"bitmap_{i}"], err_msg=f"case {i}")
        assert s.values.dtype == np.float32
        np.testing.assert_array_equal(s.values.view(np.uint32), z[f"values_{i}"].view(np.uint32))
        ref = (w.astype(np.float32) + np.float32(0.0)).astype(np.float64)
        np.testing.assert_array_equal(O.decode(s), ref)


def test_decode_block_matches_reference_goldens():
    z = _load("blocks.npz")
    s = O.encode(z["w"])
    for i in range(int(z["n"])):
        got = O.decode_block(s, tuple(z[f"rr_{i}"]), tuple(z[f"bb_{i}"]))
        np.testing.assert_array_equal(got, z[f"tile_{i}"])
    with pytest.raises(O.OracleError):
        O.decode_block(s, (0, 71), (0, 1))


def test_forward_matches_reference_goldens_bitwise():
    z = _load("forward.npz")
    for i in range(int(z["n"])):
        ads = [O.Adapter(z[f"a{j}_{i}"], z[f"b{j}_{i}"], z[f"a{j}_{i}"].shape[1], float(z[f"scale{j}_{i}"]))
               for j in range(2)]
        y = O.pipelined_forward(z[f"x_{i}"], O.encode(z[f"w_{i}"]), O.fuse(ads))
        # same f64 tile order as the reference -> bit-identical
        np.testing.assert_array_equal(y, z[f"y_{i}"], err_msg=f"case {i}")


def config1_inputs():
    """Regenerate BASELINE configs[0] inputs exactly as make_golden.py did."""
    from paper_2601_16991_b200 import synthetic
    z = _load("config1.npz")
    k, n, m = int(z["k"]), int(z["n"]), int(z["m"])
    w = synthetic.gen_weight(k, n, int(z["seed_w"])).double().numpy()
    x = synthetic.gen_x(m, k, int(z["seed_x"])).double().numpy()
    la, lb = synthetic.gen_lora(k, n, 16, int(z["seed_lora"]))
    mask = O.build_mask(w, float(z["sparsity"]))
    w_hat = np.where(mask, w, 0.0)
    ra = (z["res_a_bf16"].astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    rb = (z["res_b_bf16"].astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    ads = [O.Adapter(ra, rb, 16), O.Adapter(la.double().numpy(), lb.double().numpy(), 16, 2.0)]
    return z, w_hat, x, ads


def test_config1_oracle_matches_reference():
    z, w_hat, x, ads = config1_inputs()
    s = O.encode(w_hat)
    assert s.nnz == int(z["nnz"])
    assert hashlib.sha256(s.bitmap.tobytes()).hexdigest() == str(z["bitmap_sha256"])
    assert hashlib.sha256(s.values.tobytes()).hexdigest() == str(z["values_sha256"])
    y = O.pipelined_forward(x, s, O.fuse(ads))
    np.testing.assert_array_equal(y, z["y"])
