"""Step-level algorithmic-bytes accounting (traffic.py; SURVEY §8(d) "Time step")."""
import ctypes

from paper_2207_07098_b200 import _lib, traffic


def _acc(name, *args):
    b = [0, 0]
    traffic.account(name, args, b)
    return b


def test_models_name_real_entry_points():
    assert set(traffic.MODELS) <= set(_lib._SIGS)


def test_mgs_pass_bytes_match_the_bench_roofline():
    P = 134217728
    # w -= h v_{i-1}; <w, v_i>: w r/w, v_{i-1}, v_i, mult = 33 B/pt (bench.py MGS roofline)
    assert _acc("sf_mgs_step_f64", 1, 2, 3, 4, None, None, 5, 0, P, 6, 7, 8, None, 9) == [33 * P, 0]
    # first pass (dot + norm, read-only) and the gated second sweep
    assert _acc("sf_mgs_step_f64", 1, None, None, 4, None, None, 5, 1, P, 6, 7, 8, None, 9) == [17 * P, 0]
    assert _acc("sf_mgs_step_f64", 1, 2, 3, None, None, None, 5, 1, P, 6, 7, 8, 11, 9) == [0, 25 * P]
    # peer variant: gate is argument 17
    a = [1, 2, 3, 4, None, None, 5, 0, P, 6, 7, 8, 10, 2, 0, 1, 12, 13, 9]
    assert _acc("sf_mgs_step_peer_f64", *a) == [0, 33 * P]


def test_operator_bytes():
    E, n = 512, 8
    P = E * n ** 3
    assert _acc("sf_ax_pre_f64", 0, n, 1, 2, 3, None, 4, E, 1.0, 0.0, None, None, 0, 0)[0] == 64 * P
    assert _acc("sf_ax_pre_f64", 0, n, 1, 2, 3, 5, 4, E, 1.0, 0.0, None, None, 0, 0)[0] == 72 * P
    assert _acc("sf_ax_masked_f64", 0, n, 1, 2, 3, 4, E, 1.0, 2.0, 5, 6, 0, 0)[0] == 72 * P
    assert _acc("sf_ax_range_f64", 0, n, 1, 2, 3, None, 4, E, 10, 30, 1.0, 0.0, None, None, 0, 0)[0] \
        == 64 * 20 * n ** 3
    assert _acc("sf_deriv_f64", 0, 0, n, 1, None, 2, 3, E, 1.0, 0, 0)[0] == (8 + 72 + 24) * P
    assert _acc("sf_deriv_f64", 3, 0, n, 1, 4, 2, 3, E, 1.0, 0, 0)[0] == (24 + 24 + 72 + 24) * P
    assert _acc("sf_cdtp_f64", 0, n, 1, 2, 3, 4, E, 0, 0)[0] == 112 * P


def test_glsc3_counts_distinct_fields():
    arr = lambda *p: (ctypes.c_void_p * len(p))(*p)
    assert _acc("sf_glsc3_f64", 1, arr(100), arr(100), 7, 1000, 1, 2, 3, 0)[0] == 9 * 1000
    assert _acc("sf_glsc3_f64", 2, arr(100, 200), arr(300, 200), 7, 1000, 1, 2, 3, 0)[0] == 25 * 1000


def test_bdf_ext_counts_history_fields():
    arr = lambda *p: (ctypes.c_void_p * len(p))(*p)
    b = _acc("sf_bdf_ext_f64", 1, 2, arr(3, 4, 5), arr(6, 7, 8), arr(9, 10, 11), 0, 0, 3, 100)
    assert b[0] == 100 * 8 * (2 + 9)


def test_dssum_bytes_and_unmodeled():
    assert traffic.dssum_bytes(10, 2, 4) == 10 * 20 + 2 * 12 + 4 * 4
    b = _acc("sf_metrics_f64", 0)
    assert b == [0, 0] and "sf_metrics_f64" in traffic.UNMODELED
