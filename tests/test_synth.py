"""Input generator (synth/): seeded determinism, shard independence and the
zero-fill translate convention the oracle's sign pin relies on."""
import numpy as np
import torch

from synth import CONFIGS, config_spec, make_stack
from synth.generator import ground_truth_shifts, stripe_rows


def test_configs_match_baseline_json():
    import json, os
    bj = json.load(open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "BASELINE.json")))
    assert len(bj["configs"]) == len(CONFIGS) == 5
    shapes = [(c.T, c.m, c.n, c.dtype, c.levels, c.w) for c in CONFIGS]
    assert shapes == [(20, 64, 64, "f32", 0, 8), (1000, 256, 256, "u16", 0, 20),
                      (10000, 512, 512, "u16", 1, 16), (50000, 512, 512, "u16", 1, 32),
                      (2000, 1024, 1024, "u16", 2, 24)]


def test_deterministic_and_shard_independent():
    spec = config_spec(1, T=130)
    a = make_stack(spec, 0, 130)
    b = make_stack(spec, 60, 70)
    assert torch.equal(a.frames[60:].to(torch.int32), b.frames.to(torch.int32))
    c = make_stack(spec, 0, 130)
    assert torch.equal(a.frames.to(torch.int32), c.frames.to(torch.int32))


def test_shift_statistics():
    for c in range(5):
        spec = CONFIGS[c]
        s = ground_truth_shifts(spec)
        assert s.shape == (spec.T, 2) and np.abs(s).max() <= spec.shift_bound
        if spec.shift_kind == "walk":
            assert np.abs(np.diff(s, axis=0)).max() <= 1


def test_stripes_exact_count():
    spec = CONFIGS[3]
    r = stripe_rows(spec)
    assert (r >= 0).sum() == round(0.05 * spec.T)
    assert r.max() <= spec.m - 40


def test_zero_fill_translate_and_value_range():
    spec = config_spec(1, T=8)
    st = make_stack(spec, 0, 8)
    f = st.frames.to(torch.int32).numpy()
    assert f.max() <= 4095 and f.min() >= 0
    for k in range(8):
        dy, dx = st.shifts[k]
        if dy > 0:
            assert (f[k, :dy] == 0).all()
        if dy < 0:
            assert (f[k, dy:] == 0).all()
        if dx > 0:
            assert (f[k, :, :dx] == 0).all()
        if dx < 0:
            assert (f[k, :, dx:] == 0).all()
