"""APEX decision layer (apex_decide / apex_pipelining_threshold, CPU only) vs the
plain Algorithm 1 oracle and the SPEC.md worked examples."""
import math
import random

import pytest

from oracle import cost_model as cm
from paper_2506_03296_b200 import apex as A
from paper_2506_03296_b200 import build as B


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()


def test_threshold_matches_eq6():
    for r, want in [(0.5, 7.5), (1.0, 6.0), (1.5, 5.833333333333333), (math.sqrt(2), 2 * math.sqrt(2) + 3)]:
        assert A.apex_pipelining_threshold(1.0, r) == pytest.approx(want, rel=1e-14)
    with pytest.raises(A.ApexError):
        A.apex_pipelining_threshold(0.0, 1.0)


def test_spec_examples():
    # S:205-207 decode-only
    assert A.apex_decide(0, 1, 100, n_g=5.0, n_c=1.0, t_glinear=1.0, t_gatt=1.0)["strategy"] == "asym_pipeline"
    d = A.apex_decide(0, 1, 100, n_g=3031 / 170, n_c=1.0, t_glinear=1.0, t_gatt=1.0)   # Fig. 2b ratio 17.8
    assert d["strategy"] == "async_overlap" and d["eq6_threshold"] == 6.0
    assert A.apex_decide(0, 1, 100, n_g=2.0, n_c=2.0, t_glinear=3.0, t_gatt=0.7)["strategy"] == "asym_pipeline"
    # S:215-217 mixed: tlp = tl, tap = ta reduces to the decode-only decision
    for ng in (3.0, 5.0, 17.8):
        a = A.apex_decide(0, 1, 100, ng, 1.0, 1.0, 1.0)["strategy"]
        b = A.apex_decide(3, 1, 100, ng, 1.0, 1.0, 1.0, 1.0, 1.0)["strategy"]
        assert a == b
    # a long prefill window flips the 17.8 case to AP (CPU "has more time")
    assert A.apex_decide(3, 1, 100, 17.8, 1.0, 1.0, 1.0, 40.0, 1.0)["strategy"] == "asym_pipeline"
    # S:221-227 ratio gate (8x)
    assert A.apex_decide(0, 10, 80, 5.0, 1.0, 1.0, 1.0)["strategy"] == "asym_pipeline"
    g = A.apex_decide(0, 10, 79, 5.0, 1.0, 1.0, 1.0)
    assert g["strategy"] == "gpu_only" and g["gate_closed"]
    assert A.apex_decide(0, 10, 0, 5.0, 1.0, 1.0, 1.0)["strategy"] == "gpu_only"       # Alg. 1 line 4


def test_decide_matches_algorithm1_oracle_random():
    rnd = random.Random(0)
    for _ in range(20000):
        npf, ng_req, nc_req = rnd.choice([0, 0, 3]), rnd.randint(0, 20), rnd.choice([0, 5, 100, 400])
        args = [rnd.uniform(0.01, 50), rnd.uniform(0.01, 50), rnd.uniform(0.01, 10), rnd.uniform(0.01, 10),
                rnd.uniform(0.01, 30), rnd.uniform(0.01, 10)]
        ratio = rnd.choice([0.0, 8.0])
        want = cm.algorithm1(npf, ng_req, nc_req, *args, min_cpu_ratio=ratio)
        got = A.apex_decide(npf, ng_req, nc_req, *args, min_cpu_ratio=ratio)["strategy"]
        assert got == want


def test_decide_rejects_bad_input():
    with pytest.raises(A.ApexError):
        A.apex_decide(0, 1, 100, -1.0, 1.0, 1.0, 1.0)
    with pytest.raises(A.ApexError):
        A.apex_decide(2, 1, 100, 1.0, 1.0, 1.0, 1.0, 0.0, 1.0)
    with pytest.raises(A.ApexError):
        A.apex_decide(-1, 1, 100, 1.0, 1.0, 1.0, 1.0)
