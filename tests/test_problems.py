"""CPU checks of the seeded problem generators (problems.py) and the frozen-sequence
format (sequence.py): the product's generators draw exactly the oracle's samples, and
krecycle-sequence-v1 directories round-trip."""

from __future__ import annotations

import dataclasses

import numpy as np
import pytest


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_problem_generator_matches_oracle(name):
    from oracle import cpu_imaging as im
    from paper_2412_08264_b200.problems import CONFIGS, sample_arrays, theta0

    cfg = dataclasses.replace(CONFIGS[name], size=min(CONFIGS[name].size, 64))
    ocfg = dataclasses.replace(im.CONFIGS[name], size=cfg.size)
    for k in (0, 3):
        xt, y = sample_arrays(cfg, k)
        m, oxt = im.deblur_sample(ocfg, k)
        assert np.array_equal(xt, oxt) and np.array_equal(y, m.data.y)
    assert np.array_equal(theta0(cfg), im.deblur_theta0(ocfg))


def test_sequence_directory_roundtrip(tmp_path):
    from paper_2412_08264_b200.problems import CONFIGS
    from paper_2412_08264_b200.sequence import FORMAT_NAME, FrozenSequence, FrozenSystem, load_sequence, save_sequence

    cfg = dataclasses.replace(CONFIGS["C2"], size=8, batch=3)
    rng = np.random.default_rng(0)
    n, p = 64, 208
    systems = [FrozenSystem(i, rng.standard_normal(p), rng.standard_normal((3, n)), [5, 6, 7], 1.5 * i, 0.1, 1.0,
                            rng.standard_normal(p) if i < 2 else None) for i in range(3)]
    seq = FrozenSequence(cfg, 4, rng.standard_normal((3, n)), rng.standard_normal((3, n)), systems, {"k": "v"})
    out = save_sequence(seq, tmp_path / "seq")
    assert (out / "manifest.json").read_text().count(FORMAT_NAME) == 1
    back = load_sequence(out)
    assert back.config == cfg and back.first == 4 and back.batch == 3
    assert np.array_equal(back.x_true, seq.x_true) and np.array_equal(back.y, seq.y)
    for a, b in zip(seq.systems, back.systems):
        assert np.array_equal(a.theta, b.theta) and np.array_equal(a.x_hats, b.x_hats)
        assert a.iterations == b.iterations and a.cost == b.cost
        assert (a.theta_next is None) == (b.theta_next is None)
    (out / "manifest.json").write_text((out / "manifest.json").read_text().replace(FORMAT_NAME, "other"))
    with pytest.raises(ValueError):
        load_sequence(out)
