"""The seeded input generators: shapes, determinism and the workload structure DESIGN.md states."""
import numpy as np
import pytest

from synth import CONFIGS, make_batch, make_logits
from synth.trajectories import ACTION, PAD


@pytest.mark.parametrize("name", list(CONFIGS))
def test_batch_shapes(name):
    cfg = CONFIGS[name]
    tb = make_batch(name)
    assert tb.num_traj == cfg.num_traj
    assert tb.num_rows == cfg.num_traj * cfg.T
    assert np.all(np.diff(tb.tok_offsets) == cfg.T)
    assert np.all(tb.seg_len > 0)
    for b in range(tb.num_traj):
        s0, s1 = tb.seg_offsets[b], tb.seg_offsets[b + 1]
        assert tb.seg_len[s0:s1].sum() == cfg.T
    assert np.bincount(tb.group_id, minlength=cfg.num_groups).tolist() == [cfg.group_size] * cfg.num_groups
    tb2 = make_batch(name)
    assert np.array_equal(tb.seg_len, tb2.seg_len) and np.array_equal(tb.turn_rewards, tb2.turn_rewards)


def test_math_fractions():
    tb = make_batch("math")
    act = tb.seg_len[tb.seg_source == ACTION].sum() / tb.num_rows
    pad = tb.seg_len[tb.seg_source == PAD].sum() / tb.num_rows
    assert 0.45 < act < 0.56 and 0.30 < pad < 0.40     # 0.506 / 0.354


def test_logits_recipe():
    lg, tg = make_logits(64, 1000, ld=1008, dtype="bf16", seed=1)
    assert lg.shape == (64, 1008) and tg.dtype.is_floating_point is False
    assert float(lg[:, 1000:].float().min()) > 1e3      # padding sentinel beyond V
    a, _ = make_logits(64, 1000, dtype="bf16", seed=1)
    assert bool((a == lg[:, :1000]).all())
    assert int(((tg >= 0) & (tg < 1000)).all()) == 1
