"""Trajectory emission."""
import csv

import numpy as np
import pytest

from paper_2603_14634_b200 import pbdr as P
from paper_2603_14634_b200 import trajectory as T


def test_csv_schema_and_time_invariant(tmp_path):
    st = np.arange(2 * 3 * 13, dtype=np.float64).reshape(2, 3, 13)
    st[:, :, 3] = 1.0  # identity orientation
    path = tmp_path / "traj.csv"
    with T.TrajectoryWriter(str(path), reference=lambda t, b: ((0.0, 0.0, 0.0), 0.0)) as w:
        w.write(np.array([0.1, 0.2]), st)
        with pytest.raises(ValueError):
            w.write(np.array([0.2]), st[:1])
    rows = list(csv.reader(open(path)))
    assert ",".join(rows[0]) == T.HEADER
    assert len(rows) == 1 + 2 * 3
    assert rows[1][:3] == ["1", "0.1", "0"] and rows[4][:3] == ["2", "0.2", "0"]
    assert float(rows[1][-1]) == 0.0  # rot_err of the identity vs 0 deg
    np.testing.assert_allclose(float(rows[1][-2]), np.linalg.norm(st[0, 0, :3]))


def test_quat_angle():
    c, s = np.cos(np.pi / 8), np.sin(np.pi / 8)
    assert abs(T.quat_angle_deg([c, 0, 0, s]) - 45.0) < 1e-9


@pytest.mark.gpu
def test_device_trajectory_matches_per_frame_reads(pbdr, pyoracle):
    g = P.GeneratedScene(2)
    a = P.GpuSolver(g.desc, g.cfg)
    b = P.GpuSolver(g.desc, g.cfg)
    o = pyoracle.Oracle(g.desc, g.cfg)
    a.enable_trajectory(8)
    a.step_frames(5)
    t, st = a.drain_trajectory()
    assert st.shape == (5, g.desc.num_bodies, 13)
    np.testing.assert_allclose(np.diff(t), 1.0 / g.cfg.frame_rate, rtol=1e-9)
    for k in range(5):
        b.step_frames(1)
        assert o.step(g.cfg.substeps) == 0
        assert np.array_equal(st[k], b.read_bodies())
        assert np.array_equal(st[k], o.body_stats())
    # ring: a full ring refuses to step until drained
    a.enable_trajectory(2)
    a.step_frames(2)
    with pytest.raises(P.Error):
        a.step_frames(1)
    a.drain_trajectory()
    a.step_frames(1)


@pytest.mark.gpu
def test_record_csv(pbdr, tmp_path):
    g = P.GeneratedScene(1)
    s = P.GpuSolver(g.desc, g.cfg)
    path = tmp_path / "c1.csv"
    rows = T.record(s, 10, str(path), chunk=4)
    assert rows == 10
    lines = open(path).read().splitlines()
    assert lines[0] == T.HEADER and len(lines) == 11
