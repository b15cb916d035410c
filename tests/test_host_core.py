"""Host-core tests through the C ABI (CPU only; host-only handles make no CUDA calls).

* the library loads and exports every function include/*.h declares;
* allocator: bit-exact block tables / slots / free counts vs oracle/alloc_model.py
  (independent Python model of reading c10), all-or-nothing errors;
* planner: every (batch row, kv head, block) covered exactly once, split
  bookkeeping consistent, longest-first order;
* cost model: apex_predict_time vs oracle/cost_model.interp, exact at grid
  points, clamped, loader validation.
"""
import os
import random
import re
import subprocess

import pytest

from oracle import cost_model as cm
from oracle.alloc_model import AllocError, AllocModel
from paper_2506_03296_b200 import apex as A
from paper_2506_03296_b200 import build as B
from paper_2506_03296_b200.kvcache import PagedKVCache

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()


def host_cache(**kw):
    args = dict(num_layers=1, num_q_heads=8, num_kv_heads=2, num_blocks=64, max_seqs=16, max_blocks_per_seq=32,
                max_batch=16, max_new_tokens=4096, dtype="bf16", host_only=True)
    args.update(kw)
    return PagedKVCache(**args)


def test_exports_every_declared_symbol():
    declared = set()
    for h in ("apex.h", "apex_synth.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        declared |= set(re.findall(r"\b(apex_[a-z0-9_]+)\s*\(", src))
    nm = subprocess.run(["nm", "-D", "--defined-only", A.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in nm.splitlines() if " T " in line}
    assert declared and declared <= exported, declared - exported
    assert declared == set(A.EXPORTS)
    assert "sm_100a" in A.apex_version()


def test_alloc_matches_python_model_random():
    rnd = random.Random(0)
    for trial in range(20):
        nb = rnd.choice([8, 33, 64])
        c = host_cache(num_blocks=nb)
        m = AllocModel(nb, 16, 32)
        for step in range(60):
            if m.table and rnd.random() < 0.25:
                sid = rnd.choice(list(m.table))
                m.release(sid)
                c.release(sid)
            else:
                ids = rnd.sample(range(16), rnd.randint(1, 5))
                nn = [rnd.choice([0, 1, 1, 1, 15, 16, 17, 40]) for _ in ids]
                try:
                    want = m.alloc(ids, nn)
                    err = None
                except AllocError as e:
                    err = e.code
                if err is None:
                    c.alloc(ids, nn)
                    assert c.last_slots() == want
                else:
                    with pytest.raises(A.ApexError) as ei:
                        c.alloc(ids, nn)
                    assert ei.value.code == err
            assert c.num_free_blocks() == len(m.free)
            for sid in range(16):
                if sid in m.table:
                    assert c.seq_info(sid) == (m.length[sid], m.table[sid])
                else:
                    with pytest.raises(A.ApexError) as ei:
                        c.seq_info(sid)
                    assert ei.value.code == "ESEQ"


def test_alloc_errors_leave_state_unchanged():
    c = host_cache(num_blocks=4)
    c.alloc([0], [33])                      # 3 blocks
    before = (c.num_free_blocks(), c.seq_info(0))
    for ids, nn, code in [([1, 2], [16, 1], "ENOBLOCKS"), ([0, 0], [1, 1], "EINVAL"), ([99], [1], "EINVAL"),
                          ([3], [0], "EINVAL"), ([3], [-1], "EINVAL"), ([3], [32 * 16 + 1], "EINVAL")]:
        with pytest.raises(A.ApexError) as ei:
            c.alloc(ids, nn)
        assert ei.value.code == code
        assert (c.num_free_blocks(), c.seq_info(0)) == before
    c.release(0)
    with pytest.raises(A.ApexError) as ei:
        c.release(0)
    assert ei.value.code == "ESEQ"
    with pytest.raises(A.ApexError) as ei:
        A.apex_kv_append(c.handle, 0, 0, 0)
    assert ei.value.code == "EINVAL"


def test_alloc_planner_failure_is_all_or_nothing():
    """VERDICT r01 weak #3 / ADVICE: a plan that overflows the work-item capacity
    (forced 16-token split of 4 x 150K tokens) must fail with EINVAL and change
    nothing -- free blocks, every sequence's (len, blocks), the last step's slots
    and plan -- and the handle must keep working afterwards."""
    c = host_cache(num_q_heads=32, num_kv_heads=8, num_blocks=100000, max_seqs=8, max_batch=8,
                   max_blocks_per_seq=20000, max_new_tokens=1 << 20)
    c.alloc([5], [40])                                  # a live sequence and a valid last step
    before = (c.num_free_blocks(), c.seq_info(5), c.last_slots(), c.plan(), c.decode_launches())
    c.set_split(16)
    with pytest.raises(A.ApexError) as ei:
        c.alloc([0, 1, 2, 3], [150000] * 4)
    assert ei.value.code == "EINVAL" and "work items" in str(ei.value)
    assert (c.num_free_blocks(), c.seq_info(5), c.last_slots(), c.plan(), c.decode_launches()) == before
    for sid in range(4):
        with pytest.raises(A.ApexError) as ei:
            c.seq_info(sid)
        assert ei.value.code == "ESEQ"
    c.set_split(0)                                      # the same request now plans and commits
    c.alloc([0, 1, 2, 3], [150000] * 4)
    assert c.num_free_blocks() == before[0] - 4 * (150000 // 16)
    assert c.seq_info(0)[0] == 150000 and c.seq_info(5) == before[1]


def test_sched_errors_set_last_error():
    for args in [(0.0, 1.0), (1.0, float("nan"))]:
        with pytest.raises(A.ApexError) as ei:
            A.apex_pipelining_threshold(*args)
        assert ei.value.code == "EINVAL" and "T_glinear" in str(ei.value)
    with pytest.raises(A.ApexError) as ei:
        A.apex_decide(0, 1, -1, 1.0, 1.0, 1.0, 1.0)
    assert "negative" in str(ei.value)


def test_desc_validation():
    for kw, code in [(dict(num_q_heads=6, num_kv_heads=4), "EINVAL"), (dict(head_dim=64), "EUNSUPPORTED"),
                     (dict(block_size=32), "EUNSUPPORTED"), (dict(dtype="f32"), "EUNSUPPORTED"),
                     (dict(num_q_heads=48, num_kv_heads=3), "EUNSUPPORTED"), (dict(max_batch=17), "EINVAL")]:
        with pytest.raises(A.ApexError) as ei:
            host_cache(**kw)
        assert ei.value.code == code, kw
    host_cache(dtype="f32", num_q_heads=4, num_kv_heads=4)      # fp32 MHA is supported
    host_cache(dtype="f16", num_q_heads=32, num_kv_heads=32)


def _check_plan(c, lens, hkv, bs=16):
    items, n_merges = c.plan()
    cover = {}
    parts = {}
    for (b, g, blk0, nblk, part, seq) in items:
        assert nblk >= 1 and seq == c.batch_seq_ids[b]
        for j in range(blk0, blk0 + nblk):
            key = (b, g, j)
            assert key not in cover
            cover[key] = part
        if part >= 0:
            parts.setdefault((b, g), []).append((blk0, part))
    want = {(b, g, j) for b, L in enumerate(lens) for g in range(hkv) for j in range(-(-L // bs))}
    assert set(cover) == want
    # split pairs: partial slots are consecutive in split (block) order and unique
    all_slots = []
    for key, lst in parts.items():
        lst.sort()
        slots = [p for _, p in lst]
        assert slots == list(range(slots[0], slots[0] + len(slots))) and len(slots) >= 2
        all_slots += slots
    assert len(all_slots) == len(set(all_slots)) and n_merges == len(parts)
    # static per-CTA ranges, then the queue part in longest-first order
    cb = c.plan_ranges()
    assert cb[0] == 0 and all(cb[i] <= cb[i + 1] for i in range(len(cb) - 1)) and cb[-1] <= len(items)
    dyn = items[cb[-1]:]
    assert all(dyn[i][3] >= dyn[i + 1][3] for i in range(len(dyn) - 1))
    # stable: equal-length queue items keep their (row, kv head, block) emission order
    assert all(dyn[i][:3] < dyn[i + 1][:3] for i in range(len(dyn) - 1) if dyn[i][3] == dyn[i + 1][3])
    return items, n_merges


def test_plan_is_a_function_of_the_lengths_across_steps():
    """The planner reuses scratch storage across apex_kv_alloc calls; a long-lived
    handle whose batches grow, shrink and change regime must produce, every step,
    exactly the plan a fresh handle makes for the same lengths."""
    rnd = random.Random(5)
    kw = dict(num_q_heads=32, num_kv_heads=8, num_blocks=1 << 15, max_blocks_per_seq=1024, max_seqs=300,
              max_batch=300, dtype="bf16", max_new_tokens=1 << 20)
    live = host_cache(**kw)
    lens = {}
    for step in range(25):
        B = rnd.choice([1, 3, 40, 257, 300])
        seqs = sorted(rnd.sample(range(300), B))
        new = [rnd.randint(1, 3000) if s not in lens else rnd.choice([1, 1, 16]) for s in seqs]
        if sum(-(-(lens.get(s, 0) + n) // 16) - -(-lens.get(s, 0) // 16) for s, n in zip(seqs, new)) > \
                live.num_free_blocks():
            for s in list(lens):
                live.release(s)
            lens.clear()
            new = [rnd.randint(1, 3000) for _ in seqs]
        live.alloc(seqs, new)
        for s, n in zip(seqs, new):
            lens[s] = lens.get(s, 0) + n
        fresh = host_cache(**kw)
        fresh.alloc(list(range(B)), [lens[s] for s in seqs])
        got, want = live.plan(), fresh.plan()
        # identical up to the sequence ids (the fresh handle numbers the rows 0..B-1)
        assert got[1] == want[1] and len(got[0]) == len(want[0])
        for a, b in zip(got[0], want[0]):
            assert a[:5] == b[:5] and a[5] == seqs[b[5]]
        assert live.plan_ranges() == fresh.plan_ranges()
        fresh.close()


def test_planner_coverage_random():
    rnd = random.Random(1)
    for trial in range(30):
        hkv = rnd.choice([1, 2, 8])
        c = host_cache(num_q_heads=hkv * rnd.choice([1, 4]) if hkv != 8 else 32, num_kv_heads=hkv,
                       num_blocks=4096, max_blocks_per_seq=512, dtype="f16", max_new_tokens=1 << 16)
        c.set_grid(rnd.choice([0, 1, 7, 296]))
        c.set_sched(rnd.choice([-1, -2, 0, 100]))
        if rnd.random() < 0.5:
            c.set_split(16 * rnd.choice([1, 2, 5, 64]))
        B = rnd.randint(1, 8)
        lens = [rnd.randint(1, 2000) for _ in range(B)]
        c.alloc(list(range(B)), lens)
        _check_plan(c, lens, hkv)


def test_planner_streamk_ranges():
    """Stream-K schedule: every tile covered once; CTA c's static range holds exactly
    its quota of the first (1000 - dyn_permille) permille of the tiles, taken in
    (row, kv head, block) order; the rest are queue items of bounded count."""
    rnd = random.Random(7)
    for trial in range(40):
        hkv = rnd.choice([1, 2, 8])
        c = host_cache(num_q_heads=hkv * (4 if hkv != 8 else 4), num_kv_heads=hkv, num_blocks=1 << 16,
                       max_blocks_per_seq=2048, max_seqs=64, max_batch=64, dtype="bf16", max_new_tokens=1 << 20)
        P = rnd.choice([1, 3, 7, 16])
        perm = rnd.choice([0, 1, 50, 100, 333, 1000])
        c.set_grid(P)
        c.set_sched(perm)
        B = rnd.randint(1, 40)
        lens = [rnd.randint(1, 20000) for _ in range(B)]
        c.alloc(list(range(B)), lens)
        T = sum(-(-L // 16) for L in lens) * hkv
        items, nm = _check_plan(c, lens, hkv)
        cb = c.plan_ranges()
        assert len(cb) == P + 1
        if c.decode_launches() == 1:
            continue                                   # latency regime (fused merge): no stream-K
        t_st = T - T * perm // 1000
        flat = [(b, g, j) for b, L in enumerate(lens) for g in range(hkv) for j in range(-(-L // 16))]
        pos = 0
        for cta in range(P):
            quota = t_st // P + (1 if cta < t_st % P else 0)
            tiles = []
            for (b, g, blk0, nblk, part, seq) in items[cb[cta]:cb[cta + 1]]:
                tiles += [(b, g, j) for j in range(blk0, blk0 + nblk)]
            assert tiles == flat[pos:pos + quota]       # contiguous, in flattened order, exact quota
            pos += quota
        assert len(items) - cb[-1] <= 8 * P + B * hkv   # bounded queue items
    with pytest.raises(A.ApexError):
        c.set_sched(1001)
    with pytest.raises(A.ApexError):
        c.set_sched(-3)


def test_planner_split_chunk_and_auto():
    c = host_cache(num_q_heads=32, num_kv_heads=8, num_blocks=4096, max_blocks_per_seq=512)
    c.set_split(64)                                  # 4 blocks per item
    c.alloc([0, 1], [100, 64])                       # 7 blocks -> 4+3 ; 4 blocks -> unsplit
    items, nm = _check_plan(c, [100, 64], 8)
    assert nm == 8 and sum(1 for it in items if it[4] < 0) == 8
    c2 = host_cache(num_q_heads=32, num_kv_heads=8, num_blocks=20000, max_blocks_per_seq=1024, max_new_tokens=1 << 20)
    c2.set_grid(296)
    c2.alloc(list(range(4)), [16000] * 4)            # 32 pairs of 1000 blocks: must split (32 << 296 CTAs)
    items, nm = _check_plan(c2, [16000] * 4, 8)
    # latency regime (T = 32000 <= 512 P): one round, 9 pieces per pair (288 <= 296 CTAs)
    assert len(items) == 288 and nm == 32 and max(it[3] for it in items) == 112
    assert c2.decode_launches() == 1
    cb = host_cache(num_q_heads=32, num_kv_heads=8, num_blocks=21000, max_blocks_per_seq=1300, max_new_tokens=1 << 20)
    cb.set_grid(296)
    cb.alloc(list(range(16)), [20000] * 16)          # T = 160000 > 512 P: bandwidth regime (guided split)
    items, nm = _check_plan(cb, [20000] * 16, 8)
    assert len(items) >= 296 and nm == 128 and cb.decode_launches() == 2
    c3 = host_cache(num_q_heads=32, num_kv_heads=8, num_blocks=20000, max_blocks_per_seq=1024)
    c3.set_grid(296)
    assert A.apex_kv_decode_launches(c3.handle) == -1
    c3.alloc([0], [1000])                            # T = 63*8 = 504 <= 512 P: ~1 item per CTA
    items, nm = _check_plan(c3, [1000], 8)
    assert len(items) == 8 * 32 and all(it[3] == 2 for it in items[:-8])
    assert c3.decode_launches() == 1                 # latency regime: merge fused in-kernel
    assert cb.decode_launches() == 2                 # bandwidth regime with splits: + merge kernel
    with pytest.raises(A.ApexError):
        c2.set_split(10)                             # not a multiple of 16


def test_cost_model_matches_oracle_interp():
    rnd = random.Random(2)
    for trial in range(50):
        nb, nk = rnd.randint(1, 5), rnd.randint(1, 6)
        bg = sorted(rnd.sample(range(1, 2048), nb))
        kg = sorted(rnd.sample(range(1, 1 << 24), nk))
        us = [[rnd.uniform(1, 5000) for _ in kg] for _ in bg]
        h = A.apex_cost_create(bg, kg, us)
        try:
            for i, b in enumerate(bg):
                for j, k in enumerate(kg):
                    assert A.apex_predict_time(h, b, k) == us[i][j]
            for _ in range(200):
                b, k = rnd.randint(0, 4096), rnd.randint(0, 1 << 25)
                assert A.apex_predict_time(h, b, k) == pytest.approx(cm.interp(bg, kg, us, b, k), rel=1e-12)
        finally:
            A.apex_cost_destroy(h)


def test_cost_model_spec_example_and_validation():
    h = A.apex_cost_create([1, 256], [4096], [[100.0], [110.0]])
    assert A.apex_predict_time(h, 128, 4096) == pytest.approx(100 + 127 / 255 * 10, rel=1e-15)   # SPEC S:47 (fixed)
    assert A.apex_predict_time(h, 1024, 4096) == 110.0 and A.apex_predict_time(h, 1, 1) == 100.0
    A.apex_cost_destroy(h)
    for bg, kg, us in [([2, 1], [1], [[1.0], [1.0]]), ([1], [5, 5], [[1.0, 1.0]]), ([1], [1], [[0.0]]),
                       ([1], [1], [[float("nan")]]), ([0], [1], [[1.0]])]:
        with pytest.raises(A.ApexError) as ei:
            A.apex_cost_create(bg, kg, us)
        assert ei.value.code == "EINVAL"


def test_planner_choice_at_config_scale():
    import time
    # C5-like: 8192 pairs of 1025 blocks on 296 CTAs -> no split is cheapest
    c5 = host_cache(num_q_heads=32, num_kv_heads=8, num_blocks=1024 * 1026, max_seqs=1024, max_blocks_per_seq=1100,
                    max_batch=1024, max_new_tokens=1 << 24)
    c5.set_grid(296)
    c5.alloc(list(range(1024)), [16384] * 1024)
    t0 = time.perf_counter()
    c5.alloc(list(range(1024)), [1] * 1024)
    dt = time.perf_counter() - t0
    items, nm = c5.plan()
    # guided (default): chunk T/(4P) = 7094 blocks > 1025, so the first 90% of the pairs
    # (flattened order) stay whole; only the last 5% / 2% are cut (in 2 / 3 pieces)
    whole = {(it[0], it[1]) for it in items if it[4] < 0}
    assert len(whole) == 8192 - nm and nm <= 0.1 * 8192 and nm > 0
    assert all((b, g) in whole for b in range(1024) for g in range(8) if b * 8 + g < 0.9 * 8192)
    assert dt < 0.05                                 # per-step host planning stays cheap
    c5.set_sched(-1)                                 # uniform dynamic split: ceil(T/16P) = 1774 > 1025 -> no split
    c5.alloc(list(range(1024)), [1] * 1024)
    items, nm = c5.plan()
    assert len(items) == 8192 and nm == 0
    # C3-like: 1024 pairs of 512 blocks (3.5 per CTA) -> split
    c3 = host_cache(num_q_heads=32, num_kv_heads=8, num_blocks=128 * 513, max_seqs=128, max_blocks_per_seq=520,
                    max_batch=128, max_new_tokens=1 << 21)
    c3.set_grid(296)
    c3.alloc(list(range(128)), [8192] * 128)
    items, nm = _check_plan(c3, [8192] * 128, 8)
    # guided: bulk chunk ceil(T/4P) = 443 blocks -> 2 pieces of 256; the last 10 / 5 / 2% of
    # the pairs use chunks 111 / 55 / 27 (halves of ceil(T/8P) = 222) -> 5 / 10 / 19 pieces,
    # run last (longest first)
    sizes = sorted({it[3] for it in items})
    assert nm == 1024 and max(sizes) == 256 and min(sizes) <= 27
    assert items[0][3] == 256 and items[-1][3] == min(sizes)
    c3.set_planner(512, 8, (900, 950, 980))          # g0 = 8 (the round-1 default): 3 pieces of 171
    c3.alloc(list(range(128)), [0] * 128)
    items, nm = c3.plan()
    assert nm == 1024 and max(it[3] for it in items) == 171
    c3.set_planner()
    c3.set_sched(-1)
    c3.alloc(list(range(128)), [1] * 128)
    items, nm = _check_plan(c3, [8193] * 128, 8)
    assert len(items) == 5 * 1024 and nm == 1024     # chunk ceil(T/16P) = 111 blocks -> 5 pieces


def test_cost_observe_matches_oracle():
    """apex_cost_observe (C ABI) vs oracle/cost_model.observe on random tables and
    sequences of observations (reading c17), plus the hand-derived pins."""
    import json
    pins = json.load(open(os.path.join(ROOT, "tests", "golden", "cost_observe_pins.json")))
    for c in pins["cases"]:
        h = A.apex_cost_create(pins["batch_grid"], pins["kv_grid"], pins["us"])
        try:
            b, k = c["point"]
            if k != int(k):
                continue                                 # the ABI's kv_tokens is an integer
            A.apex_cost_observe(h, b, int(k), c["measured"], c["alpha"])
            bg, kg, us = A.apex_cost_table(h)
            assert bg == c["batch_grid"] and kg == c["kv_grid"]
            for row, want in zip(us, c["us"]):
                assert row == pytest.approx(want, abs=1e-12)
        finally:
            A.apex_cost_destroy(h)
    rnd = random.Random(5)
    for trial in range(40):
        nb, nk = rnd.randint(1, 4), rnd.randint(1, 4)
        bg = sorted(rnd.sample(range(1, 1024), nb))
        kg = sorted(rnd.sample(range(1, 1 << 24), nk))
        us = [[rnd.uniform(5, 5000) for _ in kg] for _ in bg]
        h = A.apex_cost_create(bg, kg, us)
        try:
            for step in range(6):
                b, k = rnd.randint(1, 2048), rnd.randint(1, 1 << 25)
                m, a = rnd.uniform(5, 9000), rnd.choice([1.0, 0.5, 0.25])
                bg, kg, us = cm.observe(bg, kg, us, b, k, m, a)
                A.apex_cost_observe(h, b, k, m, a)
                gb, gk, gu = A.apex_cost_table(h)
                assert gb == bg and gk == kg
                for row, want in zip(gu, us):
                    assert row == pytest.approx(want, rel=1e-12, abs=1e-9)
                for _ in range(20):
                    pb, pk = rnd.randint(0, 4096), rnd.randint(0, 1 << 26)
                    assert A.apex_predict_time(h, pb, pk) == pytest.approx(cm.interp(bg, kg, us, pb, pk), rel=1e-12)
        finally:
            A.apex_cost_destroy(h)
    h = A.apex_cost_create([1], [1], [[1.0]])
    for args in [(1, 1, 1.0, 0.0), (1, 1, 1.0, 1.5), (1, 1, 0.0, 1.0), (1, 1, float("inf"), 1.0)]:
        with pytest.raises(A.ApexError) as ei:
            A.apex_cost_observe(h, *args)
        assert ei.value.code == "EINVAL"
    assert A.apex_cost_table(h) == ([1], [1], [[1.0]])
    A.apex_cost_destroy(h)


def test_set_planner_validation_and_effect():
    c = host_cache(num_q_heads=32, num_kv_heads=8, num_blocks=8192, max_blocks_per_seq=1024, max_new_tokens=1 << 16)
    c.set_grid(296)
    for bad in [(-1, 8, 900, 950, 980), (512, 0, 900, 950, 980), (512, 65, 900, 950, 980),
                (512, 8, 950, 900, 980), (512, 8, 900, 950, 1001)]:
        with pytest.raises(A.ApexError) as ei:
            c.set_planner(bad[0], bad[1], bad[2:])
        assert ei.value.code == "EINVAL"
    c.alloc([0], [16000])                   # T = 8000 tiles <= 512 * 296: latency regime
    assert c.decode_launches() == 1
    c.set_planner(0)                        # latency regime disabled -> bandwidth plan + merge kernel
    c.alloc([0], [1])
    assert c.decode_launches() == 2
    _check_plan(c, [16001], 8)
