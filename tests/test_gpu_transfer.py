"""The reference-shaped state transfer and the simulation clock through the
C-ABI: pbdr_gpu_write_particles / read_particles (fp64, the caller's particle
order, converted and permuted on the device) and pbdr_gpu_set_time.

write_particles re-anchors the body sums and drops the warm-start rotations,
so after a write the next step equals the step of a handle created from the
written state, bit for bit (the old host path raced a legacy-stream
memset against the handle's stream and left the anchors stale)."""
import numpy as np
import pytest

from paper_2603_14634_b200 import pbdr as P

pytestmark = pytest.mark.gpu


def _scene_from_state(g, pos, vel):
    src = P.scene_with_programs(g, [P.ForceProgram()] * g.num_bodies)
    src.position[:] = pos
    src.velocity[:] = vel
    src.programs = None
    src.desc.programs = None
    return src


@pytest.mark.parametrize("cid,scale", [(2, 0), (3, 24), (5, 6)])
def test_write_particles_equals_fresh_handle(pbdr, cid, scale):
    g = P.GeneratedScene(cid, scale=scale)
    a = P.GpuSolver(g.desc, g.cfg)
    a.step_frames(30)  # warm-start rotations and anchors now differ from create
    pos, vel = a.read_particles()
    # caller order round trip: the fp64 read returns the fp32 state exactly
    p4, v4 = a.read_f32()
    assert np.array_equal(np.sort(pos[:, 0]), np.sort(p4[:, 0].astype(np.float64)))
    a.write_particles(pos, vel)
    a.set_time(0)
    fresh = _scene_from_state(g, pos, vel)
    b = P.GpuSolver(fresh.desc, g.cfg)
    np.testing.assert_array_equal(a.debug_anchor(), b.debug_anchor())
    assert not a.debug_rquat().any()
    a.step_frames(2)
    b.step_frames(2)
    pa, va = a.read_f32()
    pb, vb = b.read_f32()
    assert np.array_equal(pa, pb) and np.array_equal(va, vb)


def test_write_particles_partial_and_order(pbdr):
    # A permuted particle order (body_indices not the identity) round-trips.
    rng = np.random.default_rng(3)
    g = P.GeneratedScene(2)
    n = g.num_particles
    perm = rng.permutation(n)
    x = g.positions()[perm]
    v = g.velocities()[perm]
    inv = np.argsort(perm)
    offs = g.body_offsets()
    idx = inv[np.arange(n)].astype(np.int32)  # body k's particles, in the new order
    sc = P.ArrayScene(position=x, velocity=v, inv_mass=g.array("inv_mass", n)[perm],
                      radius=g.array("radius", n)[perm], body_offsets=offs,
                      rest_offsets=g.array("rest_offsets", 3 * n), total_mass=g.array("total_mass", g.num_bodies),
                      rest_com=g.array("rest_com", 3 * g.num_bodies), body_indices=idx)
    s = P.GpuSolver(sc.desc, g.cfg)
    pos, vel = s.read_particles()
    np.testing.assert_array_equal(pos, x.astype(np.float32).astype(np.float64))
    np.testing.assert_array_equal(vel, v.astype(np.float32).astype(np.float64))
    v2 = vel * 0.5
    s.write_particles(None, v2)  # velocities only: positions, anchors untouched
    _, vel2 = s.read_particles()
    np.testing.assert_array_equal(vel2, v2)


def test_set_time_opens_force_windows(pbdr):
    # A force window [t0, t1) far into the run: only a clock seeded at t0
    # applies it (stateless pbdr::step calls pass the scene time this way).
    g = P.GeneratedScene(1)
    dt = 1.0 / (g.cfg.frame_rate * g.cfg.substeps)
    prog = P.ForceProgram((5.0, 0.0, 0.0), (0.0, 0.0, 0.0), 100 * dt, 101 * dt, 0, 0)
    sc = P.scene_with_programs(g, [prog])
    late = P.GpuSolver(sc.desc, g.cfg)
    late.set_time(100)
    assert late.get_time() == 100
    early = P.GpuSolver(sc.desc, g.cfg)
    late.step(1)
    early.step(1)
    assert late.get_time() == 101 and early.get_time() == 1
    vl = late.read_bodies()[0, 7:10]
    ve = early.read_bodies()[0, 7:10]
    np.testing.assert_allclose(vl[0] - ve[0], 5.0 * dt, rtol=1e-3)  # dP = F dt, M = 1 kg
