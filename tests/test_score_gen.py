"""Score generation on the device: numpy's PCG64 uniform
streams (default_rng(seed).uniform, the reference's synth.py:156-195 draws and
the benchmark's per-channel streams) reproduced bit for bit by
``ab_scores_generate``.

CPU: a pure-Python restatement of the generator the kernel implements (LCG
step, XSL-RR output, O(log n) jump-ahead) checked against numpy itself — it
pins the constants and the jump algorithm.  GPU: the kernel's output equals
numpy's, f32 and f64."""

import numpy as np
import pytest

from paper_2306_15685_b200 import synth

M128 = (1 << 128) - 1
MULT = 0x2360ED051FC65DA44385DF649FCCF645


def step(state, inc):
    state = (state * MULT + inc) & M128
    hi, lo = state >> 64, state & ((1 << 64) - 1)
    x, rot = hi ^ lo, hi >> 58
    return state, ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)


def advance(state, inc, delta):
    acc_mult, acc_plus, cur_mult, cur_plus = 1, 0, MULT, inc
    while delta:
        if delta & 1:
            acc_mult = acc_mult * cur_mult & M128
            acc_plus = (acc_plus * cur_mult + cur_plus) & M128
        cur_plus = (cur_mult + 1) * cur_plus & M128
        cur_mult = cur_mult * cur_mult & M128
        delta >>= 1
    return (acc_mult * state + acc_plus) & M128


def test_restatement_matches_numpy():
    for seed in ([7, 0], [7, 1023], 12345, [11, 3, 1]):
        st = synth.pcg64_streams([seed])[0]
        state = (int(st[0]) << 64) | int(st[1])
        inc = (int(st[2]) << 64) | int(st[3])
        raw = np.random.default_rng(seed).bit_generator.random_raw(300)
        s = state
        for k in range(300):
            s, x = step(s, inc)
            assert x == int(raw[k])
        # jump-ahead lands where stepping does
        for k in (0, 1, 63, 64, 200):
            _, x = step(advance(state, inc, k), inc)
            assert x == int(raw[k])
        u = np.random.default_rng(seed).uniform(0.0, 6.0, 50)
        s = state
        for k in range(50):
            s, x = step(s, inc)
            assert 0.0 + 6.0 * ((x >> 11) * (1.0 / 9007199254740992.0)) == u[k]


@pytest.mark.gpu
def test_device_channel_scores_bit_exact():
    chans = [0, 5, 1023]
    got = synth.device_channel_scores(7, chans, 9, 2000).cpu().numpy()
    for i, c in enumerate(chans):
        assert np.array_equal(got[i], synth.channel_scores(7, c, 9, 2000))


@pytest.mark.gpu
def test_device_uniform_f64_offset_ragged_length():
    # synth_score_matrix's draw: noise + rng.uniform(0.0, 0.1, size)
    seeds = [[3, i] for i in range(5)]
    n = 1000 * 3 + 7  # not a multiple of the per-thread chunk
    got = synth.device_uniform(seeds, n, 0.0, 0.1, offset=5.0, dtype="float64").cpu().numpy()
    for i, sd in enumerate(seeds):
        assert np.array_equal(got[i], 5.0 + np.random.default_rng(sd).uniform(0.0, 0.1, n))
