"""Bodies larger than one iteration CTA (more than 2048 particles, up to
32768): each runs on a thread-block cluster (k_iteration_big, DSMEM partial
sums into the leader CTA) with the same pinned reduction tree as the tiled
kernel, so the results stay bit-exact against the oracle. These are the
resolution-study bodies (run_resolution_study; PAPER.md section
V-B: box and bunny at increasing sphere counts)."""
import numpy as np
import pytest

from paper_2603_14634_b200 import pbdr as P

pytestmark = pytest.mark.gpu


def _rot(seed):
    q = np.random.default_rng(seed).normal(size=4)
    w, x, y, z = q / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def _box(nx, ny, nz, s=0.02, centre=(0.0, 0.0, 1.0), seed=None):
    g = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1).reshape(-1, 3)
    x = (g - (np.array([nx, ny, nz]) - 1) / 2.0) * s
    if seed is not None:
        x = x @ _rot(seed).T
    return x + np.array(centre)


def _spin(x, w, v=(0.0, 0.0, 0.0)):
    c = x.mean(0)
    return np.cross(np.asarray(w, dtype=np.float64), x - c) + np.asarray(v)


def assert_same(a, b, what):
    if not np.array_equal(a, b):
        diff = np.abs(a.astype(np.float64) - b.astype(np.float64))
        raise AssertionError(f"{what}: {np.count_nonzero(diff)} differ, max {diff.max():.3g}")


def _compare(pyoracle, sc, cfg, frames):
    gpu = P.GpuSolver(sc.desc, cfg)
    orc = pyoracle.Oracle(sc.desc, cfg)
    assert gpu.info.tile_kp == orc.tile_kp == 8  # a big body forces the KP = 8 tree
    gpu.step_frames(frames)
    assert orc.step(frames * cfg.substeps) == 0
    gp, gv = gpu.read_f32()
    op, ov = orc.read_f32()
    assert np.abs(gp - op).max() <= 1e-5
    assert_same(gp, op, "positions")
    assert_same(gv, ov, "velocities")
    assert_same(gpu.read_bodies(), orc.body_stats(), "body stats")
    return gpu, orc


def _single_box(n_axis, seed=1, programs=False):
    x = _box(n_axis, n_axis, n_axis, centre=(0.0, 0.0, 0.02 * n_axis), seed=seed)
    v = _spin(x, (0.5, -1.0, 2.0), (0.3, 0.0, -0.5))
    sc = P.ArrayScene(**P.rigid_body_arrays([x], 0.01, [2.0], velocities=[v]),
                      ground=P.Plane((0, 0, 0), (0, 0, 1), 0.5))
    if programs:
        sc = P.scene_with_programs(sc, [P.ForceProgram((1.0, 0.0, 0.0), (0.0, 0.0, 0.2), 0.0, float("inf"), 0, 0)])
    return sc


@pytest.mark.parametrize("n_axis", [13, 16, 21])  # 2197 (2 CTAs), 4096 (2), 9261 (5)
def test_single_big_body_bit_exact(pbdr, pyoracle, n_axis):
    # One body per scene: all iterations of a substep in one cluster launch,
    # state held in the cluster's shared memory; ground contact with friction.
    _compare(pyoracle, _single_box(n_axis), P.solver_cfg(frame_rate=240.0), 4)


def test_big_body_torque_program_bit_exact(pbdr, pyoracle):
    # distribute_wrench of a big body (looping-CTA torque prepass).
    _compare(pyoracle, _single_box(16, seed=4, programs=True), P.solver_cfg(frame_rate=240.0), 3)


def test_largest_body_bit_exact(pbdr, pyoracle):
    # 32^3 = 32768 particles: 128 warps, a 16-CTA (non-portable) cluster.
    _compare(pyoracle, _single_box(32, seed=2), P.solver_cfg(frame_rate=240.0), 1)


def _mixed_scene():
    # Two big bodies (4800 and 2500 particles: clusters of 3, the second
    # leaves a CTA idle) under a rain of 27-particle bodies: contacts between
    # big and small bodies, so both kernels run every iteration.
    bodies, vels = [], []
    big = _box(20, 20, 12, centre=(0.0, 0.0, 0.125), seed=None)
    bodies.append(big)
    vels.append(np.zeros_like(big))
    big2 = _box(10, 10, 25, centre=(0.6, 0.0, 0.26), seed=None)
    bodies.append(big2)
    vels.append(np.zeros_like(big2))
    rng = np.random.default_rng(5)
    for k in range(12):
        c = (rng.uniform(-0.15, 0.15), rng.uniform(-0.15, 0.15), 0.3 + 0.07 * k)
        x = _box(3, 3, 3, centre=c, seed=10 + k)
        bodies.append(x)
        vels.append(_spin(x, rng.normal(size=3), (0.0, 0.0, -1.0)))
    masses = [3.0, 1.5] + [0.05] * 12
    return P.ArrayScene(**P.rigid_body_arrays(bodies, 0.01, masses, velocities=vels),
                        ground=P.Plane((0, 0, 0), (0, 0, 1), 0.4))


def test_mixed_big_and_small_bodies_with_contacts(pbdr, pyoracle):
    gpu, orc = _compare(pyoracle, _mixed_scene(), P.solver_cfg(frame_rate=60.0), 6)
    # Contacts did happen: some small body was stopped (free fall from -1 m/s
    # would reach about -2 m/s after 0.1 s).
    stats = gpu.read_bodies()
    assert (stats[2:, 9] / 0.05).max() > -0.5


@pytest.mark.parametrize("variant", ["pbd", "legacy_fixed", "per_substep", "linear_only"])
def test_big_body_solver_variants(pbdr, pyoracle, variant):
    cfg = {"pbd": P.pbd_cfg(frame_rate=240.0),
           "legacy_fixed": P.solver_cfg(frame_rate=240.0, velocity_update=0),
           "per_substep": P.solver_cfg(frame_rate=240.0, momentum_frequency=1),
           "linear_only": P.solver_cfg(frame_rate=240.0, angular_momentum_fix=False)}[variant]
    _compare(pyoracle, _mixed_scene(), cfg, 2)


def test_big_bodies_in_slab_roles(pbdr):
    # Slab mode with every body owned runs the same launches on the same
    # bodies: identical to the whole-scene path.
    sc = _mixed_scene()
    cfg = P.solver_cfg(frame_rate=60.0)
    a = P.GpuSolver(sc.desc, cfg)
    b = P.GpuSolver(sc.desc, cfg)
    b.set_roles(np.full(sc.num_bodies, 2, dtype=np.int8))
    for _ in range(3):
        a.step_frames(1)
        b.step_frames(1)
    pa, va = a.read_f32()
    pb, vb = b.read_f32()
    assert_same(pa, pb, "positions")
    assert_same(va, vb, "velocities")

