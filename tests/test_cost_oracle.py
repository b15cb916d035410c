"""Pins for oracle/cost_model.py (CPU only): SPEC/PAPER worked values and Eq5<=>Eq6."""
import json
import math
import os
import random

import pytest

from oracle import cost_model as cm

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cost_model_pins.json")))


def test_interp_1d_spec_examples():
    g = G["interp_1d"]
    for x, want in g["cases"]:
        got = cm.interp(g["grid"], [1], [[u] for u in g["us"]], x, 1)
        assert got == pytest.approx(want, rel=1e-15, abs=1e-12)


def test_interp_exact_at_grid_points_and_clamped():
    bg, kg = [1, 4, 16], [512, 4096, 32768]
    us = [[3.0 + i * 7 + j * 11.5 + i * j for j in range(3)] for i in range(3)]
    for i, b in enumerate(bg):
        for j, k in enumerate(kg):
            assert cm.interp(bg, kg, us, b, k) == us[i][j]
    assert cm.interp(bg, kg, us, 0, 1) == us[0][0]
    assert cm.interp(bg, kg, us, 99, 10**9) == us[2][2]
    assert cm.interp(bg, kg, us, 99, 512) == us[2][0]


def test_interp_bilinear_reproduces_bilinear_functions():
    # a bilinear function f(x,y) = a + bx + cy + dxy is reproduced exactly inside each cell
    f = lambda x, y: 2.0 + 0.5 * x - 0.25 * y + 0.125 * x * y
    bg, kg = [1.0, 3.0, 10.0], [0.0, 8.0, 20.0]
    us = [[f(x, y) for y in kg] for x in bg]
    rnd = random.Random(3)
    for _ in range(200):
        x, y = rnd.uniform(1, 10), rnd.uniform(0, 20)
        assert cm.interp(bg, kg, us, x, y) == pytest.approx(f(x, y), rel=1e-12)


def test_eq6_paper_values():
    for c in G["eq6"]["cases"]:
        r = c["t_gatt_over_t_glinear"]
        assert cm.eq6_threshold(1.0, r) == pytest.approx(c["threshold"], rel=1e-14)
        assert cm.eq6_threshold(3.0, 3.0 * r) == pytest.approx(c["threshold"], rel=1e-14)  # scale-free
    # paper: on [0.5, 1.5] the threshold is at most ~7.5, so CPU must be >= ~13% of GPU
    worst = max(cm.eq6_threshold(1.0, 0.5 + i / 1000) for i in range(1001))
    assert worst == pytest.approx(7.5) and 1 / worst == pytest.approx(0.1333, abs=1e-3)
    assert min(cm.eq6_threshold(1.0, 0.5 + i / 10000) for i in range(10001)) >= 2 * math.sqrt(2) + 3 - 1e-12


def test_eq5_equivalent_to_eq6_random():
    rnd = random.Random(0)
    bad = 0
    for _ in range(100000):
        tl, ta = rnd.uniform(0.01, 10), rnd.uniform(0.01, 10)
        ng, nc = rnd.uniform(0.01, 100), rnd.uniform(0.01, 100)
        ratio, thr = ng / nc, cm.eq6_threshold(tl, ta)
        if abs(ratio - thr) < 1e-9 * thr:
            continue
        bad += cm.eq5_holds(ng, nc, tl, ta) != (ratio < thr)
    assert bad == 0


def test_eq1_to_eq4_and_fig_b_rates():
    assert cm.t_gpuonly(2.0, 3.0) == 5.0 and cm.t_overlap(2.0, 3.0) == 7.0
    assert cm.n_gtotal(4.0, 3.0) == 12.0 and cm.n_ctotal(0.5, 2.0, 3.0) == 3.5
    f = G["fig_b_rates"]
    assert f["kv_tokens"] / f["gpu_us"] == pytest.approx(f["n_g_tokens_per_us"], rel=1e-15)
    assert f["cpu_us"] / f["gpu_us"] == pytest.approx(f["ng_over_nc"], rel=1e-15)


# ---- online recalibration (reading c17)

GO = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cost_observe_pins.json")))


def test_observe_hand_derived_pins():
    for c in GO["cases"]:
        b, k = c["point"]
        bg, kg, us = cm.observe(GO["batch_grid"], GO["kv_grid"], GO["us"], b, k, c["measured"], c["alpha"])
        assert bg == c["batch_grid"] and kg == c["kv_grid"], c["what"]
        for row, want in zip(us, c["us"]):
            assert row == pytest.approx(want, abs=1e-12), c["what"]


def test_observe_properties():
    """Invariants of reading c17 on random tables: the input table is untouched; after one
    step the prediction at the point is pred + alpha*e; predictions outside the point's
    cell (and everywhere, for the grid-line insertion alone) are unchanged."""
    rnd = random.Random(11)
    for _ in range(200):
        nb, nk = rnd.randint(1, 4), rnd.randint(1, 4)
        bg = sorted(rnd.sample(range(1, 500), nb))
        kg = sorted(rnd.sample(range(1, 10 ** 6), nk))
        us = [[rnd.uniform(1, 1000) for _ in kg] for _ in bg]
        snap = [row[:] for row in us]
        b, k = rnd.randint(0, 600), rnd.randint(0, 2 * 10 ** 6)
        m, a = rnd.uniform(1, 2000), rnd.choice([1.0, 0.5, 0.1])
        pred = cm.interp(bg, kg, us, b, k)
        bg2, kg2, us2 = cm.observe(bg, kg, us, b, k, m, a)
        assert us == snap
        assert cm.interp(bg2, kg2, us2, b, k) == pytest.approx(pred + a * (m - pred), rel=1e-9, abs=1e-9)
        # probes whose cell shares no corner with the point's cell keep their predictions
        def corners(x, y):
            i, _ = cm._axis(bg2, x)
            j, _ = cm._axis(kg2, y)
            return {(a, c) for a in (i, min(i + 1, len(bg2) - 1)) for c in (j, min(j + 1, len(kg2) - 1))}
        mine = corners(b, k)
        for _ in range(20):
            pb, pk = rnd.randint(0, 600), rnd.randint(0, 2 * 10 ** 6)
            if corners(pb, pk) & mine:
                continue
            assert cm.interp(bg2, kg2, us2, pb, pk) == pytest.approx(cm.interp(bg, kg, us, pb, pk), rel=1e-9)
    with pytest.raises(ValueError):
        cm.observe([1], [1], [[1.0]], 1, 1, 1.0, 0.0)
    with pytest.raises(ValueError):
        cm.observe([1], [1], [[1.0]], 1, 1, -1.0, 1.0)


def test_algorithm1_direct_pins():
    """oracle.cost_model.algorithm1 pinned by itself on SPEC.md
    S:201-239 examples and hand-evaluated Eq5 sides (Alg. 1)."""
    a1 = cm.algorithm1
    # S:205 N_G/N_C = 5 < Eq6 threshold 6 (T_gatt = T_glinear): lhs (5+3)/3 = 2.67 > rhs 5/2 = 2.5
    assert a1(0, 1, 100, 5.0, 1.0, 1.0, 1.0) == "asym_pipeline"
    # S:206 Fig. 2b ratio 3031/170 = 17.83 > 6: lhs (17.83+3)/3 = 6.94 < rhs 8.91
    assert a1(0, 1, 100, 3031 / 170, 1.0, 1.0, 1.0) == "async_overlap"
    # exactly at the Eq6 threshold (N_G/N_C = 6): lhs (6+3)/3 = 3 == rhs 6/2 = 3, strict ">" -> AO
    assert a1(0, 1, 100, 6.0, 1.0, 1.0, 1.0) == "async_overlap"
    # S:207 N_C = N_G -> AP for any positive times (ratio 1 < min threshold 2*sqrt(2)+3)
    for tl, ta in [(0.1, 9.0), (3.0, 0.7), (1.0, 1.0)]:
        assert a1(0, 1, 100, 2.0, 2.0, tl, ta) == "asym_pipeline"
    # S:215 mixed with T_glinear_pref = T_glinear, T_gatt_pref = T_gatt == decode-only
    for ng in (3.0, 5.0, 17.8):
        assert a1(3, 1, 100, ng, 1.0, 1.0, 1.0, 1.0, 1.0) == a1(0, 1, 100, ng, 1.0, 1.0, 1.0)
    # S:216 a long prefill window: lhs (17.8 + 42)/3 = 19.93 > rhs 8.9 -> AP
    assert a1(3, 1, 100, 17.8, 1.0, 1.0, 1.0, 40.0, 1.0) == "asym_pipeline"
    # S:217 N_C -> 0 in the mixed branch -> AO
    assert a1(3, 1, 100, 17.8, 1e-12, 1.0, 1.0, 40.0, 1.0) == "async_overlap"
    # S:221-227 ratio gate: 80 >= 8*10 passes; 79 closes; no CPU requests -> GPU-only
    assert a1(0, 10, 80, 5.0, 1.0, 1.0, 1.0) == "asym_pipeline"
    assert a1(0, 10, 79, 5.0, 1.0, 1.0, 1.0) == "gpu_only"
    assert a1(0, 10, 0, 5.0, 1.0, 1.0, 1.0) == "gpu_only"
    assert a1(0, 10, 79, 5.0, 1.0, 1.0, 1.0, min_cpu_ratio=0.0) == "asym_pipeline"
