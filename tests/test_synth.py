"""Input generator + NSPL interchange; parameter accounting."""
import math

import numpy as np
import pytest

import synth


def test_parameter_count_is_99():
    assert synth.PARAMS_PER_PRIM == 99                        # P:394 "99 parameters in total"
    assert 8 * 3 + 8 + 8 + 1 == 41                            # P:751 "41 parameters from its 8-neuron MLP"
    sc = synth.make_scene(0, 10)
    assert sc.records().shape == (10, 99)


def test_paper_init_ranges():
    sc = synth.make_scene(1, 5000, variant="paper")
    bound = math.sqrt(6 / 8) / 30
    assert abs(bound - 0.028868) < 1e-6
    assert np.abs(sc.w2).max() <= bound and np.abs(sc.w2).max() > 0.95 * bound
    assert np.abs(sc.w1).max() <= 1 / 3 + 1e-7                # P:393 W1 ~ U(-1/3, 1/3)


def test_nspl_roundtrip(tmp_path):
    sc = synth.make_scene(2, 100)
    p = tmp_path / "s.nspl"
    synth.save_nspl(sc, p)
    assert p.stat().st_size == 32 + 99 * 4 * 100
    sc2 = synth.load_nspl(p)
    for f in ("centers", "rotations", "scales", "w1", "b1", "w2", "b2", "sh"):
        assert np.array_equal(getattr(sc, f), getattr(sc2, f))
    raw = p.read_bytes()
    (tmp_path / "t.nspl").write_bytes(raw[:-7])
    with pytest.raises(ValueError, match="truncated"):
        synth.load_nspl(tmp_path / "t.nspl")
    (tmp_path / "m.nspl").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(ValueError, match="magic"):
        synth.load_nspl(tmp_path / "m.nspl")


def test_configs_shapes_and_determinism():
    a, ca, _ = synth.make_config("C1")
    b, cb, _ = synth.make_config("C1")
    assert a.n == 256 and ca[0].width == 128 and np.array_equal(a.w1, b.w1)
    _, c4, _ = synth.make_config("C4", n=100)
    assert len(c4) == 64
    for c in c4:
        R = c.R_wc.astype(np.float64)
        assert np.allclose(R.T @ R, np.eye(3), atol=1e-6)
