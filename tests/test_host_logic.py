"""CPU: the product library's host logic (schedules, SDA controller, RNG
jump-ahead, data permutation, teacher data) against the oracle, bit for bit,
and the C-ABI surface declared in include/dasmc_gpu.h."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_abi_exports_every_declared_symbol(product):
    hdr = open(os.path.join(ROOT, "include", "dasmc_gpu.h")).read()
    names = set(re.findall(r"\b(dasmc_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 25
    lib = product.load()
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_batch_size_tables_bit_exact(product, oracle):
    rng = np.random.default_rng(1)
    cases = [(k, 500, 500, 200, 60000, 1, -1) for k in range(5)]
    cases += [(2, 200, 100, 50, 2000, 1, 40), (3, 1000, 1000, 300, 60000, 5, 300), (3, 100, 100, 50, 2000, 1, -1)]
    for _ in range(30):
        N = int(rng.integers(2, 5000))
        Cb = int(rng.integers(1, N + 1))
        kap = int(rng.integers(1, N + 1))
        K = int(rng.integers(1, 300))
        cases.append((int(rng.integers(0, 5)), Cb, kap, K, N, int(rng.integers(1, 6)), int(rng.integers(-1, K))))
    for kind, c0, kap, K, N, per, sw in cases:
        names = ["constant", "full_batch", "ctr", "linear", "automated"]
        cfg = product.ScheduleConfig(names[kind], c0, kap, K, N, per, sw)
        got = [product.batch_size(cfg, k) for k in range(K)]
        exp = [oracle.batch_size(kind, c0, kap, K, N, per, sw, k) for k in range(K)]
        assert got == exp, (kind, c0, kap, K, N, per, sw)
    with pytest.raises(ValueError):
        product.batch_size(product.ScheduleConfig("constant", 5, 5, 10, 100), 10)
    with pytest.raises(ValueError):
        product.batch_size(product.ScheduleConfig("sda", 5, 5, 10, 100), 0)


def test_sda_controller_bit_exact(product, oracle):
    rng = np.random.default_rng(2)
    for _ in range(200):
        beta = float(rng.uniform(0.01, 1.0))
        step = float(rng.choice([-1.0, 1.0]) * rng.uniform(0.1, 3))
        denom = float(rng.choice([0.0, rng.normal() * 10]))
        assert product.sda_beta_step(beta, step, denom) == oracle.sda_beta_step(beta, step, denom)
    for J in (2, 3, 17, 128):
        pre, blk = rng.normal(size=J) * 50, rng.normal(size=J) * 20
        lw = rng.normal(size=J) * 3
        lw[0] = -np.inf
        np.testing.assert_array_equal(product.sda_moments_from(pre, blk, lw), oracle.sda_moments_from(pre, blk, lw))
    cfg = product.ScheduleConfig("sda", 100, 100, 50, 1000)
    st = product.sda_init(cfg, 0.1, 1.0)
    ost = [st.beta, st.entropy_step, st.beta_reset, st.prefix_end, st.block_end, st.total_n, st.stage, st.terminal]
    for _ in range(300):
        m6 = rng.normal(size=6) * 5
        m6[2] = abs(m6[2])
        st = product.sda_advance_with(cfg, st, m6)
        ost = oracle.sda_advance_with(100, 1000, ost, m6)
        assert [st.beta, st.entropy_step, st.prefix_end, st.block_end, st.stage, st.terminal] == \
            [ost[0], ost[1], ost[3], ost[4], ost[6], ost[7]]
    assert st.terminal == 1 and st.prefix_end == 1000


def test_rng_jump_ahead_matches_sequential_stream(product, oracle):
    lib = product.load()
    for key in (0, oracle.fork_key(7, 2, 5, 3), 2**63 + 12345):
        ref = oracle.rng_u64(key, 5000)
        for skip in (0, 1, 2, 63, 255, 256, 2047, 2048, 4096, 4990):
            out = np.empty(8, dtype=np.uint64)
            assert lib.dasmc_rng_skip(key, skip, 8, out.ctypes.data_as(C.POINTER(C.c_uint64))) == 0
            assert np.array_equal(out, ref[skip:skip + 8]), (key, skip)


def test_shuffle_permutation_matches(product, oracle):
    for seed, n in ((0, 100), (123, 2000), (2**40, 7)):
        assert np.array_equal(product.shuffle_permutation(seed, n), oracle.shuffle_perm(seed, n))


def test_teacher_data_matches(product, oracle):
    for layers, act, kind in (([8, 4, 3], "relu", 0), ([12, 6, 4], "tanh", 1), ([64, 32, 10], "tanh", 0)):
        spec = product.NetSpec(layers, act)
        X, y = product.make_teacher_data(spec, 300, kind, 11, 2, threads=4)
        Xo, yo = oracle.make_teacher(layers, 0 if act == "relu" else 1, 300, kind, 11, 2)
        assert np.array_equal(X, Xo.astype(np.float32))
        assert np.array_equal(y, yo)


def test_invalid_arguments_raise(product):
    lib = product.load()
    d = product.NetSpec([4, 0, 2]).desc()
    h = C.c_void_p()
    X = np.zeros((4, 4), dtype=np.float32)
    y = np.zeros(4, dtype=np.int32)
    rc = lib.dasmc_gpu_create(C.byref(d), X.ctypes.data_as(C.POINTER(C.c_float)),
                              y.ctypes.data_as(C.POINTER(C.c_int32)), 4, 8, 0, 0, C.byref(h))
    assert rc == -1 and b"layer sizes" in lib.dasmc_last_error()


def test_redraw_rows_bit_exact(product, oracle):
    """draw_batch_rows (runner.hpp:531-542): partial Fisher-Yates with fork(kRedraw, k)."""
    M64 = (1 << 64) - 1
    for seed, k, n, count in ((0, 0, 100, 10), (7, 13, 1000, 1000), (3, 2, 57, 1)):
        u = iter(int(v) for v in oracle.rng_u64(oracle.fork_key(seed, 6, k, 0), 4 * count + 64))

        def below(b):  # rng.hpp:66-73
            limit = M64 - (M64 % b)
            while True:
                x = next(u)
                if x < limit:
                    return x % b
        order = list(range(n))
        for i in range(count):
            j = i + below(n - i)
            order[i], order[j] = order[j], order[i]
        assert list(product.redraw_rows(seed, k, n, count)) == order[:count]
