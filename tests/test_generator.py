"""Generator pins (CPU): splitmix64 reference vectors, value lattice, RNE rounding."""
import numpy as np

import synth


def test_splitmix64_reference_sequence():
    # Vigna's splitmix64.c seeded with 0 emits these first three values
    g = 0x9E3779B97F4A7C15
    want = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    assert [synth.splitmix64_int(k * g % 2**64) for k in range(3)] == want
    arr = synth.splitmix64(np.array([k * g % 2**64 for k in range(3)], dtype=np.uint64))
    assert [int(x) for x in arr] == want


def test_values_on_lattice_and_range():
    x = synth.gen_f32(1, 3, np.arange(1000), 2, 5, np.arange(128)[:, None])
    assert x.dtype == np.float32 and x.min() >= -2 and x.max() < 2
    assert np.all((x.astype(np.float64) * 2**22) == np.round(x.astype(np.float64) * 2**22))
    assert abs(x.var() - 4 / 3) < 0.02 and abs(x.mean()) < 0.02
    assert np.array_equal(synth.gen_f32(0, 0, 1, 2, 3, 4, amp=8), 8 * synth.gen_f32(0, 0, 1, 2, 3, 4))


def test_keys_distinct_fields():
    k = synth.make_key(2, 63, 65535, 127, (1 << 18) - 1, 255)
    assert int(k) == (1 << 56) | ((1 << 55) - 1)   # tensor=2 -> bit 56; every other field all-ones
    a = synth.gen_f32(1, 0, 0, 0, np.arange(5000), 0)
    assert len(np.unique(a)) > 4900


def test_rne_rounding_bf16_and_f16():
    x = np.array([1.0, 1.0 + 2**-8, 1.0 + 3 * 2**-8, -2.0, 1.0 + 2**-11, 1.0 + 3 * 2**-11],
                 dtype=np.float32)
    bf = synth.f32_to_bf16_bits(x)
    # 1+2^-8 is a tie -> even (1.0); 1+3*2^-8 tie -> up to 1+2^-6
    assert list(bf[:4]) == [0x3F80, 0x3F80, 0x3F82, 0xC000]
    h = synth.f32_to_f16_bits(x)
    assert list(h[[0, 4, 5]]) == [0x3C00, 0x3C00, 0x3C02]
