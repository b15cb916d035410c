"""Pins for oracle/alloc_model.py (CPU only): hand-worked sequences + conservation."""
import random

import pytest

from oracle.alloc_model import AllocError, AllocModel


def test_hand_worked_sequence():
    m = AllocModel(num_blocks=4, max_seqs=8, max_blocks_per_seq=4)
    assert m.alloc([0], [17]) == list(range(16)) + [16]        # blocks 0,1
    assert m.table[0] == [0, 1]
    assert m.alloc([3, 0], [1, 15]) == [32] + list(range(17, 32))   # seq 3 -> block 2; seq0 fills blk 1
    assert m.alloc([0], [1]) == [48]                          # pos 32 -> block 3
    with pytest.raises(AllocError) as e:
        m.alloc([5], [1])
    assert e.value.code == "ENOBLOCKS"
    m.release(0)                                               # pushes 3,1,0 -> pops 0,1,3
    assert m.alloc([5], [40]) == list(range(0, 32)) + list(range(48, 56))
    assert m.table[5] == [0, 1, 3]


def test_all_or_nothing_and_errors():
    m = AllocModel(num_blocks=3, max_seqs=4, max_blocks_per_seq=8)
    m.alloc([0], [16])
    snap = (list(m.free), {k: list(v) for k, v in m.table.items()}, dict(m.length))
    with pytest.raises(AllocError) as e:
        m.alloc([1, 2], [16, 17])                              # needs 3 > 2 free
    assert e.value.code == "ENOBLOCKS"
    assert snap == (m.free, m.table, m.length)
    for args in (([0, 0], [1, 1]), ([9], [1]), ([1], [0]), ([1], [8 * 16 + 1])):
        with pytest.raises(AllocError) as e:
            m.alloc(*args)
        assert e.value.code == "EINVAL"
    with pytest.raises(AllocError) as e:
        m.release(3)
    assert e.value.code == "ESEQ"


def test_conservation_random():
    rnd = random.Random(1)
    m = AllocModel(num_blocks=64, max_seqs=16, max_blocks_per_seq=32)
    for _ in range(2000):
        if m.table and rnd.random() < 0.2:
            m.release(rnd.choice(list(m.table)))
        else:
            ids = rnd.sample(range(16), rnd.randint(1, 4))
            try:
                slots = m.alloc(ids, [rnd.randint(1, 40) for _ in ids])
                assert len(set(slots)) == len(slots)
            except AllocError as e:
                assert e.code in ("ENOBLOCKS", "EINVAL")
        assert len(m.free) + m.held() == 64
        held = [b for t in m.table.values() for b in t]
        assert len(set(held)) == len(held) and not set(held) & set(m.free)
