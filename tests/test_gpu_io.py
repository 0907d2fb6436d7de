"""GPU: the report kernel (moco_mean_image) and the CLI end to end."""
import numpy as np
import pytest
import torch

from paper_1506_06039_b200 import Plan, cli, io
from synth import config_spec, make_stack
from tests import paper_forms as pf

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def test_mean_image_exact():
    """Two frames [[0]] and [[2]] -> [[1]]; identical frames -> that frame; random u16 and
    f32 stacks against numpy's fp64 mean (u16: exact sums, one division)."""
    a = torch.tensor([[[0]], [[2]]], dtype=torch.int32).to(torch.uint16).to(DEV)
    assert io.mean_image(a).cpu().tolist() == [[1.0]]
    rng = np.random.default_rng(6)
    x = rng.integers(0, 4096, (37, 30, 41)).astype(np.uint16)
    got = io.mean_image(torch.from_numpy(x).to(DEV)).cpu().numpy()
    assert np.array_equal(got, x.astype(np.int64).sum(0) / 37.0)
    same = np.repeat(x[:1], 5, 0)
    assert np.array_equal(io.mean_image(torch.from_numpy(same).to(DEV)).cpu().numpy(), x[0].astype(np.float64))
    y = rng.random((9, 12, 13)).astype(np.float32)
    np.testing.assert_allclose(io.mean_image(torch.from_numpy(y).to(DEV)).cpu().numpy(), y.astype(np.float64).mean(0),
                               rtol=1e-12)


def test_cli_align_drifting_stack(tmp_path):
    """Noise-free drifting stack (exact integer translates of the first frame, |s|,|t| <=
    20, 128x128, auto config: levels 0, w = 42) through the CLI: the shift CSV recovers
    every applied shift, f = 0 on every frame, and the corrected stack's mean image has
    more variance than the raw one's."""
    spec = config_spec(1, m=128, n=128, T=1, n_blobs=60)
    tp = make_stack(spec, 0, 1).template.numpy()
    rng = np.random.default_rng(7)
    T = 50
    truth = rng.integers(-20, 21, (T, 2))
    truth[0] = 0
    fr = np.stack([pf.translate_zero_fill(tp, int(dy), int(dx)) for dy, dx in truth]).astype(np.uint16)
    src, dst = str(tmp_path / "in.tif"), str(tmp_path / "out.tif")
    csv, mb, ma = str(tmp_path / "s.csv"), str(tmp_path / "mb.tif"), str(tmp_path / "ma.tif")
    io.save_stack(fr, src)
    assert cli.main(["align", "--input", src, "--output", dst, "--shifts-csv", csv, "--mean-before", mb,
                     "--mean-after", ma]) == 0
    sh, fm, flags = io.read_shift_log(csv)
    assert sh.tolist() == truth.tolist() and (fm == 0).all()
    out = io.load_stack(dst)
    assert out.shape == fr.shape
    for k in (0, 7, 33):
        assert np.array_equal(out[k], pf.translate_zero_fill(fr[k], -int(truth[k, 0]), -int(truth[k, 1]))
                              * (pf.translate_zero_fill(np.ones_like(fr[k]), -int(truth[k, 0]), -int(truth[k, 1])) > 0))
    g = io.mean_image_variance_gain(io.load_stack(mb)[0], io.load_stack(ma)[0], border=21)
    assert g >= 1.2, g


def test_mean_image_gain_on_c2_stack():
    """Figure 2's claim made quantitative on the C2 generator's drifting stack (walk to
    +-28 px, Poisson noise): variance of the corrected mean image >= 1.2 x the raw one's."""
    spec = config_spec(2, T=400)
    st = make_stack(spec, 0, 400, device=DEV)
    p = Plan(512, 512, 16, 1, "u16", 12, device=0)
    p.set_template(st.template)
    _, _, co, _ = p.align(st.frames, corrected=True)
    g = io.mean_image_variance_gain(io.mean_image(st.frames).cpu().numpy(), io.mean_image(co).cpu().numpy(),
                                    border=30)
    assert g >= 1.2, g
