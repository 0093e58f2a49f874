"""The CUDA path against the INDEPENDENT fp64 oracle (oracle/pbdr_oracle64.cpp)
at the north_star tolerances -- no bit-exactness expected or used.

The fp32 oracle (pbdr_oracle.cpp) is bit-exact with the GPU because it
replays the GPU's reduction trees and shares its pinned header; these tests
catch anything the two could get wrong together. The fp64 oracle shares only
the semantic pins (P1-P6): plain fp64 sums, the reference's cold
scaled-Newton polar and SPD pseudo-inverse.

north_star bars checked here (tolerances written in the asserts):
* per-particle positions after one step (a frame of 10 substeps) within
  1e-5 m, all five configs (C3/C4/C5 scaled; C3 and C4 also at full size);
* single-body com / orientation trajectories over 1000 steps within 1e-3
  relative (config 1, a seeded tumbling cube that lands on the ground);
* chaotic pile aggregates (pile com, kinetic energy) within 1% through the
  landing, settled pile height within 2% (config 2).
"""
import numpy as np
import pytest

from paper_2603_14634_b200 import pbdr as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cid,scale", [(1, 0), (2, 0), (3, 24), (4, 3), (5, 6), (3, 0), (4, 0)])
def test_one_step_within_1e5(pbdr, pyoracle, cid, scale):
    g = P.GeneratedScene(cid, scale=scale)
    gpu = P.GpuSolver(g.desc, g.cfg)
    o = pyoracle.Oracle64(g.desc, g.cfg)
    gpu.step_frames(1)
    assert o.step(g.cfg.substeps) == 0
    gp, _ = gpu.read_particles()
    op, _ = o.read_particles()
    err = np.abs(gp - op).max()
    assert err <= 1e-5, f"C{cid}: max |dx| = {err:.3g} m"
    np.testing.assert_allclose(gpu.read_bodies()[:, 0:3], o.body_stats()[:, 0:3], atol=1e-5)


def _quat_dist(a, b):
    # rotation-invariant distance of unit quaternions (q ~ -q)
    return np.minimum(np.linalg.norm(a - b, axis=-1), np.linalg.norm(a + b, axis=-1))


def test_single_body_1000_steps(pbdr, pyoracle):
    g = P.GeneratedScene(1)
    gpu = P.GpuSolver(g.desc, g.cfg)
    o = pyoracle.Oracle64(g.desc, g.cfg)
    gpu.enable_trajectory(1000)
    gpu.step_frames(1000)
    _, traj = gpu.drain_trajectory()
    worst_c, worst_q = 0.0, 0.0
    for f in range(1000):
        assert o.step(g.cfg.substeps) == 0
        s = o.body_stats()[0]
        gc, gq = traj[f, 0, 0:3], traj[f, 0, 3:7]
        worst_c = max(worst_c, np.linalg.norm(gc - s[0:3]) / max(np.linalg.norm(s[0:3]), 1e-3))
        worst_q = max(worst_q, _quat_dist(gq, s[3:7]))
    assert worst_c <= 1e-3, f"com relative error {worst_c:.3g}"
    assert worst_q <= 1e-3, f"orientation (unit quaternion) error {worst_q:.3g}"


def test_pile_aggregates_within_1pct(pbdr, pyoracle):
    # Config 2 through its landing (frame 60: first impacts under way): pile com
    # and kinetic energy within 1%. Later the pile is chaotic: two correct
    # implementations with different rounding diverge body by body (measured
    # between the fp32 and fp64 oracles: KE 18.7 vs 21.5 J at frame 120, com x
    # 6.1 vs 2.6 cm at frame 1000 -- DESIGN.md section 8), so the settled pile
    # is compared on what stays deterministic in aggregate: its height (the
    # potential energy) within 2% and a vanishing kinetic energy.
    g = P.GeneratedScene(2)
    gpu = P.GpuSolver(g.desc, g.cfg)
    o = pyoracle.Oracle64(g.desc, g.cfg)
    m = 1.0 / g.array("inv_mass", g.num_particles)

    def aggregates(p, v):
        return (p * m[:, None]).sum(0) / m.sum(), 0.5 * (m * (v ** 2).sum(1)).sum(), (m * 9.81 * p[:, 2]).sum()

    gpu.step_frames(60)
    assert o.step(60 * g.cfg.substeps) == 0
    (cg, kg, _), (co, ko, _) = aggregates(*gpu.read_particles()), aggregates(*o.read_particles())
    assert np.abs(cg - co).max() <= 0.01 * np.abs(co).max()
    assert abs(kg - ko) <= 0.01 * ko
    gpu.step_frames(420)
    assert o.step(420 * g.cfg.substeps) == 0
    (cg, kg, pg), (co, ko, po) = aggregates(*gpu.read_particles()), aggregates(*o.read_particles())
    assert abs(pg - po) <= 0.02 * po
    assert kg < 5e-3 * po and ko < 5e-3 * po
