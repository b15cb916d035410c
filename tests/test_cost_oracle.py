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
