"""Pins of the RACE scheduling oracle (§4.3-§5) and the roofline model (§3)."""
import csv
import json
import math
import os

import numpy as np
import pytest

from oracle import perfmodel as pm
from oracle import race

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _table():
    with open(os.path.join(GOLD, "paper_table2_table3.csv")) as f:
        rows = [r for r in csv.reader(l for l in f if not l.startswith("#"))]
    hdr = rows[0]
    return [dict(zip(hdr, r)) for r in rows[1:]]


def _ex():
    with open(os.path.join(GOLD, "paper_worked_examples.json")) as f:
        return json.load(f)


# ------------------------------------------------------------- perf model (§3)
def test_table3_reproduction():
    """Table 3 cols 3-4 from Table 2: alpha_opt = 1/NNZR and
    I_SpMV(alpha_opt) by Eq. 2; starred SKX entries = 1/SymmNNZR (Eq. 4)."""
    rows = _table()
    assert len(rows) == 31
    for r in rows:
        nnzr = int(r["nnz"]) / int(r["nrows"])
        assert abs(float(r["nnzr"]) - nnzr) < 6e-3
        a = float(r["alpha_opt"])
        # printed alpha_opt agrees with nrows/nnz of Table 2 to ~1e-7 relative ...
        assert abs(a * nnzr - 1.0) < 2e-7
        # ... and column 4 is Eq. 2 at NNZR = 1/alpha_opt, to the last printed digit
        assert abs(pm.intensity_spmv(1.0 / a, a) / float(r["I_opt"]) - 1.0) < 1e-15
        if r["skx_star"] == "1":  # starred: alpha_SymmSpMV = 1/SymmNNZR (Eq. 4)
            assert abs(float(r["alpha_symm_skx"]) * pm.symm_nnzr(1.0 / a) - 1.0) < 1e-15


def test_spin26_roofline_and_alpha():
    e = _ex()["spin26_roofline"]
    assert round(pm.alpha_from_traffic_spmv(e["bytes_per_nnz_ivb"], e["nnzr"]), 3) == e["alpha_ivb"]
    # 16.36 B inverts to 0.3664; the paper prints 0.367 (Table 3: 0.367034) -> 1e-3 tolerance
    assert abs(pm.alpha_from_traffic_spmv(e["bytes_per_nnz_skx"], e["nnzr"]) - e["alpha_skx"]) < 1e-3
    I_ivb = pm.intensity_symmspmv(e["nnzr"], e["alpha_symm_ivb_table3"])
    I_skx = pm.intensity_symmspmv(e["nnzr"], e["alpha_symm_skx_table3"])
    lo, hi = pm.roofline(I_ivb, e["bw_ivb_copy"]), pm.roofline(I_ivb, e["bw_ivb_load"])
    assert abs(lo - e["gf_ivb"][0]) < 0.006 and abs(hi - e["gf_ivb"][1]) < 0.011
    lo, hi = pm.roofline(I_skx, e["bw_skx_copy"]), pm.roofline(I_skx, e["bw_skx_load"])
    assert abs(lo - e["gf_skx"][0]) < 0.006 and abs(hi - e["gf_skx"][1]) < 0.006
    # limits: Eq. 3 with alpha = 1/SymmNNZR, NNZR -> inf gives 4/12
    assert abs(pm.intensity_symmspmv(1e12, 0.0) - 4.0 / 12.0) < 1e-9
    assert pm.symm_nnzr(14.0) == 7.5 and pm.symm_nnzr(1.0) == 1.0


def test_min_bytes_is_eq3_at_alpha_opt():
    """bytes_min = nnz_u / I_SymmSpMV(1/SymmNNZR) * 4  (Eq. 3 at the optimal alpha)."""
    for n, nnz_full in ((4096, 20224), (2097152, 55742968), (134217728, 937951232)):
        nnz_u = (nnz_full + n) // 2
        symm = nnz_u / n
        nnzr = 2 * symm - 1  # Eq. 4 inverted
        I = pm.intensity_symmspmv(nnzr, 1.0 / symm)
        bytes_eq3 = 4 * nnz_u / I
        assert abs(pm.symmspmv_min_bytes(n, nnz_u) - 4 - bytes_eq3) / bytes_eq3 < 1e-12


# ------------------------------------------------------------- §4.4.3 epsilon windows
def test_eps_window_paper_example():
    e = _ex()["eps_window_stencil16"]
    lw = e["level_sizes"]
    assert sum(lw) == 256
    W = race.eps_aggregate(lw, e["nthreads"], e["k"], e["eps"])
    f, l, b = W[0]
    assert (l - f, b) == (e["first_window_levels"], e["first_window_threads"])
    assert sum(lw[f:l]) / (256 / 8) == e["first_window_weight"]
    # T_0(4), T_0(5) = third window: four levels, weight 54/32, two threads
    f, l, b = W[2]
    assert l - f == e["pair2_levels"] and sum(lw[f:l]) == e["pair2_weight_num"] and b == e["pair2_threads"]
    assert sum(b for _, _, b in W) == e["threads_total"]
    assert sum(1 for _, _, b in W if b == 2) == e["pairs_with_two_threads"]
    # windows tile the levels and hold >= 2k levels
    assert W[0][0] == 0 and W[-1][1] == len(lw)
    assert all(W[i][1] == W[i + 1][0] for i in range(len(W) - 1))
    assert all(l - f >= 2 * e["k"] for f, l, _ in W)


def test_eps_degenerate():
    assert race.eps_aggregate([5, 5, 5], 4, 2, 0.8) == [(0, 3, 1)]
    assert race.eps_aggregate([], 4, 2, 0.8) == []
    W = race.eps_aggregate([1] * 40, 1, 2, 0.5)
    assert sum(b for *_, b in W) >= 1 and W[-1][1] == 40


# ------------------------------------------------------------- Alg. 4 invariants
def _groups_from_windows(lw, W, k):
    T, wk = [W[0][0]], []
    for f, l, b in W:
        m = race.split_window(lw, f, l, k)
        T += [m, l]
        wk += [b, b]
    return T, wk


@pytest.mark.parametrize("seed", range(6))
def test_alg4_invariants(seed):
    rng = np.random.default_rng(seed)
    L = int(rng.integers(12, 80))
    lw = [int(v) for v in rng.integers(1, 200, size=L)]
    k = 2
    T0 = [int(round(i * L / 6)) for i in range(7)]
    if any(T0[i + 1] - T0[i] < k for i in range(6)):
        pytest.skip("initial split violates k")
    T, hist = race.alg4_balance(T0, [1] * 6, lw, kmin=k)
    # terminates, variance non-increasing, >= k levels kept, same end points
    assert all(hist[i + 1] < hist[i] for i in range(len(hist) - 1))
    assert all(T[i + 1] - T[i] >= k for i in range(6))
    assert T[0] == 0 and T[-1] == L


def test_alg4_balanced_and_blocked():
    # perfectly balanced -> unchanged
    T, hist = race.alg4_balance([0, 2, 4, 6, 8], [1] * 4, [1] * 8, kmin=2)
    assert T == [0, 2, 4, 6, 8] and len(hist) == 1
    # the only shift would leave a group with < k levels -> unchanged
    T, _ = race.alg4_balance([0, 2, 4], [1, 1], [10, 10, 1, 1], kmin=2)
    assert T == [0, 2, 4]


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


@pytest.mark.parametrize("case", [0, 1])
def test_alg4_hand_traces(case):
    """Exact T_ptr after every outer iteration and the exact variances of a
    hand trace of Alg. 4 (tests/golden/alg4_hand_traces.json); case 1 has
    workers != 1, which pins reading R14's per-colour mean by value."""
    g = _gold("alg4_hand_traces.json")
    c = g["cases"][case]
    trace = []
    T, hist = race.alg4_balance(g["T_ptr0"], c["workers"], g["level_work"], kmin=2, trace=trace)
    assert trace == c["T_trace"]
    assert T == c["T_final"]
    want = c.get("var_hist") or [n / d for n, d in c["var_hist_num_den"]]
    assert len(hist) == len(want)
    assert all(abs(h - w) <= 1e-15 * max(1.0, abs(w)) for h, w in zip(hist, want))


def test_alg4_stencil16_ten_groups():
    """on the 16x16 stencil with ten level groups the end
    groups get more levels (fewer rows per level), the middle groups keep 2."""
    g = _gold("alg4_hand_traces.json")["stencil16_ten_groups"]
    lw, ng = g["level_sizes"], g["n_groups"]
    L = len(lw)
    T0 = [int(math.floor(i * L / ng + 0.5)) for i in range(ng + 1)]
    T, hist = race.alg4_balance(T0, [1] * ng, lw, kmin=2)
    nl = [T[i + 1] - T[i] for i in range(ng)]
    assert T[0] == 0 and T[-1] == L and min(nl) >= 2
    assert nl[0] > 2 and nl[-1] > 2
    assert all(v == 2 for v in nl[2:-2])
    # levels per group do not increase from either end toward the middle
    assert all(nl[i] >= nl[i + 1] for i in range(ng // 2 - 1))
    assert all(nl[-1 - i] >= nl[-2 - i] for i in range(ng // 2 - 1))
    assert hist[-1] < hist[0]


def test_split_window_hand_cases():
    """Reading R13: the red part ends at the first level boundary where it holds
    at least half the window's work, clamped so both parts keep >= k levels."""
    lw = [1, 2, 3, 4, 5, 6]
    # cumulative 1,3,6,10,15: 2*15 >= 21 first at boundary 5, clamped to end-k = 4
    assert race.split_window(lw, 0, 6, 2) == 4
    # window [2, 6): cumulative 3, 7, 12: 2*12 >= 18 first at boundary 5, clamped to end-k = 4
    assert race.split_window(lw, 2, 6, 2) == 4
    assert race.split_window([5, 5, 5, 5], 0, 4, 2) == 2
    assert race.split_window([9, 1, 1, 1, 1, 1, 1, 1], 0, 8, 2) == 2  # heavy first level: clamp to first + k
    assert race.split_window([1, 1, 1], 0, 3, 2) == 2  # < 2k levels: first + ceil(3/2)


def test_alg4_improves_skewed_17_levels():
    """Fig. 10-like: 17 levels, 6 groups, skewed start."""
    lw = [1, 2, 3, 5, 8, 9, 10, 10, 10, 9, 8, 7, 5, 4, 3, 2, 1]
    T0 = [0, 2, 4, 6, 8, 10, 17]
    T, hist = race.alg4_balance(T0, [1] * 6, lw, kmin=2)
    assert hist[-1] < hist[0]
    assert all(T[i + 1] - T[i] >= 2 for i in range(6))


# ------------------------------------------------------------- §5 nrowsEff, eta
def test_nrows_eff_and_eta():
    assert race.nrows_eff([10, 6]) == 16
    assert race.nrows_eff([[10, 9, 12, 11], 5]) == 12 + 11 + 5  # inner {10,12}/{9,11} -> 23
    e = _ex()["eta_stencil16"]
    # the 44-row tree itself is a lost figure: its root nrowsEff (printed, 44) stands for it
    eta = race.eta(256, e["nrowsEff_root"], e["nthreads"])
    assert round(eta, 2) == e["eta"]
    assert round(eta * 8, 1) == e["speedup"]
    assert race.eta(256, [256, 0], 1) == 1.0
    assert race.eta(20, [5, 5, 5, 5], 2) == 1.0
