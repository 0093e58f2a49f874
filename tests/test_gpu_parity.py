"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on
identical seeded inputs.

north_star bars: hash-cell assignments and contact-pair sets bit-exact;
positions after one step within 1e-5 m; single-body com/orientation
trajectories over 1000 steps within 1e-3 relative; free-flight P/L conserved
within 1e-5 relative; piles' aggregates within 1%. Because both sides follow
the same pinned op order, most comparisons here are bit-exact; the
north_star tolerances are asserted as well, in the test bodies.
"""
import numpy as np
import pytest

from paper_2603_14634_b200 import pbdr as P

pytestmark = pytest.mark.gpu

# (config, scale): scaled-down configs keep the oracle within seconds.
CASES = [(1, 0), (2, 0), (3, 24), (4, 3), (5, 6)]


def pair(pyoracle, cid, scale=0, seed=0, cfg=None):
    g = P.GeneratedScene(cid, seed=seed, scale=scale)
    c = g.cfg if cfg is None else cfg
    return g, P.GpuSolver(g.desc, c), pyoracle.Oracle(g.desc, c)


def assert_same(a, b, what):
    if not np.array_equal(a, b):
        diff = np.abs(a.astype(np.float64) - b.astype(np.float64))
        idx = np.unravel_index(np.argmax(diff), diff.shape)
        raise AssertionError(f"{what}: {np.count_nonzero(diff)} differ, max {diff.max():.3g} at {idx}")


@pytest.mark.parametrize("cid,scale", CASES)
def test_prologue_bit_exact(pbdr, pyoracle, cid, scale):
    g, gpu, orc = pair(pyoracle, cid, scale)
    gpu.debug_prologue()
    orc.integrate()
    orc.candidates()
    gp, gv = gpu.read_f32()
    op, ov = orc.read_f32()
    assert_same(gp, op, "integrated positions")
    assert_same(gv, ov, "integrated velocities")
    assert_same(gpu.debug_init(), orc.read_init(), "x_init")
    # Hash-cell assignment (cell coordinates and bucket) bit-exact.
    gh, gc = gpu.debug_keys()
    oh, oc = orc.keys()
    assert_same(gc, oc, "cell coordinates")
    assert_same(gh, oh, "cell hash")
    # Onesweep output over the broadphase-filtered ("near") particles: sorted,
    # distinct slots, stable, keys equal to the particles' cell hashes.
    k, v = gpu.debug_sorted()
    assert np.all(k[1:] >= k[:-1])
    assert len(np.unique(v)) == len(v)
    same = k[1:] == k[:-1]
    assert np.all(v[1:][same] > v[:-1][same])
    assert np.array_equal(k, oh[v])
    # Contact candidate sets bit-exact (ascending slot order).
    gcnt, glst = gpu.debug_candidates()
    ocnt, olst = orc.read_candidates()
    assert_same(gcnt, ocnt, "candidate counts")
    mask = np.arange(P.NBR_CAP)[None, :] < gcnt[:, None]
    assert_same(np.where(mask, glst, -1), np.where(mask, olst, -1), "candidate lists")
    # Symmetry of the pair set.
    ii = np.repeat(np.arange(gpu.n), gcnt)
    jj = glst[mask]
    fwd = set(zip(ii.tolist(), jj.tolist()))
    assert all((j, i) in fwd for i, j in fwd)


@pytest.mark.parametrize("cid,scale", CASES)
def test_iterations_bit_exact(pbdr, pyoracle, cid, scale):
    g, gpu, orc = pair(pyoracle, cid, scale)
    gpu.debug_prologue()
    orc.integrate()
    orc.candidates()
    for it in range(g.cfg.solver_iterations):
        gpu.debug_iteration()
        orc.iteration()
        gp, gv = gpu.read_f32()
        op, ov = orc.read_f32()
        assert_same(gp, op, f"positions after iteration {it}")
        assert_same(gv, ov, f"velocities after iteration {it}")
        assert_same(gpu.debug_anchor(), orc.read_anchor(), f"anchors after iteration {it}")
        assert_same(gpu.debug_rquat(), orc.read_rquat(), f"warm-start rotations after iteration {it}")


@pytest.mark.parametrize("cid,scale", CASES)
def test_one_frame_matches_oracle(pbdr, pyoracle, cid, scale):
    g, gpu, orc = pair(pyoracle, cid, scale)
    gpu.step_frames(1)  # CUDA-graph replay of one frame (10 substeps)
    assert orc.step(g.cfg.substeps) == 0
    gp, gv = gpu.read_particles()
    op, ov = orc.read_particles()
    assert np.abs(gp - op).max() <= 1e-5  # north_star: one step within 1e-5 m
    assert np.array_equal(gp, op) and np.array_equal(gv, ov)
    assert_same(gpu.read_bodies(), orc.body_stats(), "body stats")


@pytest.mark.parametrize("kp", [2, 4, 8])
@pytest.mark.parametrize("cid,scale", [(2, 0), (3, 24), (5, 6)])
def test_tile_shapes_bit_exact(pbdr, pyoracle, kp, cid, scale):
    # Every tile shape (particles per lane, pbdr_choose_kp) reduces with its own
    # pinned tree; the oracle follows the same shape, so all stay bit-exact.
    g = P.GeneratedScene(cid, seed=0, scale=scale)
    g.desc.tile_kp = kp
    gpu = P.GpuSolver(g.desc, g.cfg)
    orc = pyoracle.Oracle(g.desc, g.cfg)
    assert gpu.info.tile_kp == orc.tile_kp >= kp
    gpu.step_frames(2)
    assert orc.step(2 * g.cfg.substeps) == 0
    gp, gv = gpu.read_f32()
    op, ov = orc.read_f32()
    assert_same(gp, op, f"kp={kp} positions")
    assert_same(gv, ov, f"kp={kp} velocities")
    assert_same(gpu.read_bodies(), orc.body_stats(), f"kp={kp} body stats")


def test_tile_shape_rule(pbdr):
    # The measured per-scene choice.
    assert P.GpuSolver(P.GeneratedScene(1).desc, P.solver_cfg()).info.tile_kp == 2


def test_graph_replay_equals_direct_substeps(pbdr):
    g = P.GeneratedScene(2)
    a = P.GpuSolver(g.desc, g.cfg)
    b = P.GpuSolver(g.desc, g.cfg)
    a.step_frames(3)
    b.step(3 * g.cfg.substeps)
    pa, va = a.read_f32()
    pb, vb = b.read_f32()
    assert np.array_equal(pa, pb) and np.array_equal(va, vb)


def test_odd_iteration_count_parity(pbdr, pyoracle):
    g = P.GeneratedScene(2)
    cfg = P.solver_cfg(frame_rate=240.0, substeps=3, solver_iterations=5)
    gpu = P.GpuSolver(g.desc, cfg)
    orc = pyoracle.Oracle(g.desc, cfg)
    gpu.step_frames(3)
    assert orc.step(9) == 0
    assert np.array_equal(gpu.read_f32()[0], orc.read_f32()[0])


@pytest.mark.parametrize("variant", ["pbd", "linear_only", "angular_only", "legacy_fixed", "per_substep"])
def test_solver_variants_bit_exact(pbdr, pyoracle, variant):
    # SolverConfig::pbd(), the Table IV ablations and MomentumFrequency
    # (scene.hpp:15, 22-25, 33-39).
    cfg = {"pbd": P.pbd_cfg(frame_rate=240.0),
           "linear_only": P.solver_cfg(frame_rate=240.0, angular_momentum_fix=False),
           "angular_only": P.solver_cfg(frame_rate=240.0, linear_momentum_fix=False),
           "legacy_fixed": P.solver_cfg(frame_rate=240.0, velocity_update=0),
           "per_substep": P.solver_cfg(frame_rate=240.0, momentum_frequency=1)}[variant]
    g = P.GeneratedScene(2)
    gpu = P.GpuSolver(g.desc, cfg)
    orc = pyoracle.Oracle(g.desc, cfg)
    gpu.step_frames(2)
    assert orc.step(2 * cfg.substeps) == 0
    gp, gv = gpu.read_f32()
    op, ov = orc.read_f32()
    assert_same(gp, op, variant + " positions")
    assert_same(gv, ov, variant + " velocities")


def _programs(nb, seed=3):
    # Mix of force-only, torque-only, force+torque, windowed and gravity-exempt
    # programs (scene.hpp:53-61); bodies with no wrench keep a null program.
    rng = np.random.default_rng(seed)
    out = []
    for b in range(nb):
        kind = b % 5
        F = tuple(rng.uniform(-5, 5, 3)) if kind in (1, 3) else (0.0, 0.0, 0.0)
        tau = tuple(rng.uniform(-0.05, 0.05, 3)) if kind in (2, 3, 4) else (0.0, 0.0, 0.0)
        t0, t1 = (0.002, 0.006) if kind == 4 else (0.0, float("inf"))
        out.append(P.ForceProgram(F, tau, t0, t1, int(kind == 2), 0))
    return out


def test_force_torque_programs_bit_exact(pbdr, pyoracle):
    # External wrench programs on the GPU path:
    # force at the com plus torque distributed as m_p * (I^-1 tau) x r_p
    # (body.cpp:126-150), inside [t_start, t_stop), gravity_exempt bodies.
    g = P.GeneratedScene(2)
    sc = P.scene_with_programs(g, _programs(g.desc.num_bodies))
    cfg = P.solver_cfg(frame_rate=240.0)
    gpu = P.GpuSolver(sc.desc, cfg)
    orc = pyoracle.Oracle(sc.desc, cfg)
    gpu.debug_prologue()
    orc.integrate()
    assert_same(gpu.read_f32()[1], orc.read_f32()[1], "velocities after the wrench integrate")
    gpu = P.GpuSolver(sc.desc, cfg)
    orc = pyoracle.Oracle(sc.desc, cfg)
    gpu.step_frames(3)
    assert orc.step(3 * cfg.substeps) == 0
    gp, gv = gpu.read_f32()
    op, ov = orc.read_f32()
    assert_same(gp, op, "positions")
    assert_same(gv, ov, "velocities")
    assert_same(gpu.read_bodies(), orc.body_stats(), "body stats")


@pytest.mark.slow
def test_c1_trajectory_1000_steps(pbdr, pyoracle):
    # north_star: single-body com / orientation over 1000 steps within 1e-3 rel.
    g, gpu, orc = pair(pyoracle, 1)
    worst_com, worst_ang = 0.0, 0.0
    for frame in range(1000):
        gpu.step_frames(1)
        assert orc.step(g.cfg.substeps) == 0
        if frame % 50 == 49 or frame == 999:
            sg, so = gpu.read_bodies()[0], orc.body_stats()[0]
            worst_com = max(worst_com, np.abs(sg[0:3] - so[0:3]).max() / max(1e-3, np.abs(so[0:3]).max()))
            d = abs(float(np.dot(sg[3:7], so[3:7])))
            worst_ang = max(worst_ang, 2 * np.arccos(min(1.0, d)))
    assert worst_com <= 1e-3 and worst_ang <= 1e-3
    assert np.array_equal(gpu.read_f32()[0], orc.read_f32()[0])


def test_free_flight_momentum_gpu(pbdr):
    # north_star: free-flight P and L conserved within 1e-5 relative over the
    # config-1 free-flight window (45 frames before the cube can reach the
    # ground), and per substep within 1e-6 max(1, |P0|)
    # over 10^4 substeps.
    g = P.GeneratedScene(1)
    cfg = P.solver_cfg(frame_rate=240.0, gravity=0.0)
    sc = P.ArrayScene(position=g.positions(), velocity=g.velocities(), inv_mass=g.array("inv_mass", 512),
                      radius=g.array("radius", 512), body_offsets=[0, 512],
                      rest_offsets=g.array("rest_offsets", 3 * 512), total_mass=[1.0],
                      rest_com=g.array("rest_com", 3), has_ground=False)
    gpu = P.GpuSolver(sc.desc, cfg)
    s0 = gpu.read_bodies()[0]
    gpu.step_frames(45)
    s1 = gpu.read_bodies()[0]
    assert np.linalg.norm(s1[7:10] - s0[7:10]) <= 1e-5 * np.linalg.norm(s0[7:10])
    assert np.linalg.norm(s1[10:13] - s0[10:13]) <= 1e-5 * np.linalg.norm(s0[10:13])
    prev = s1
    worst = 0.0
    for _ in range(100):
        gpu.step(10 * cfg.substeps)
        cur = gpu.read_bodies()[0]
        worst = max(worst, np.abs(cur[7:10] - prev[7:10]).max() / 100, np.abs(cur[10:13] - prev[10:13]).max() / 100)
        prev = cur
    assert worst <= 1e-6 * max(1.0, np.linalg.norm(s0[7:10]))


@pytest.mark.slow
def test_c2_pile_aggregates(pbdr, pyoracle):
    # north_star: chaotic piles agree on aggregates (pile com, KE) within 1%.
    g, gpu, orc = pair(pyoracle, 2)
    frames = 120
    gpu.step_frames(frames)
    assert orc.step(frames * g.cfg.substeps) == 0
    gp, gv = gpu.read_particles()
    op, ov = orc.read_particles()
    m = 1.0 / g.array("inv_mass", g.num_particles)
    com_g = (gp * m[:, None]).sum(0) / m.sum()
    com_o = (op * m[:, None]).sum(0) / m.sum()
    ke_g = 0.5 * (m * (gv ** 2).sum(1)).sum()
    ke_o = 0.5 * (m * (ov ** 2).sum(1)).sum()
    assert np.abs(com_g - com_o).max() <= 0.01 * np.abs(com_o).max()
    assert abs(ke_g - ke_o) <= 0.01 * max(ke_o, 1e-12)
    assert np.array_equal(gp, op)


def test_deterministic_reruns(pbdr):
    # identical scene + config + seed -> bit-identical trajectory.
    g = P.GeneratedScene(3, scale=64)
    a = P.GpuSolver(g.desc, g.cfg)
    b = P.GpuSolver(g.desc, g.cfg)
    a.step_frames(2)
    b.step_frames(2)
    assert np.array_equal(a.read_f32()[0], b.read_f32()[0])


def test_penetration_bound_c2(pbdr):
    # SPEC.md:341 (frame-boundary penetration <= 10% of r) on the settling pile.
    g = P.GeneratedScene(2)
    gpu = P.GpuSolver(g.desc, g.cfg)
    gpu.step_frames(240)
    p, _ = gpu.read_particles()
    r = g.array("radius", g.num_particles)
    assert (p[:, 2] - r).min() >= -0.1 * r.max()


@pytest.mark.parametrize("cid,scale,frames", [(2, 0, 60), (3, 250, 200), (4, 8, 60), (5, 6, 60)])
def test_replay_contact_rich_state(pbdr, pyoracle, cid, scale, frames):
    # Differential replay: advance the GPU into a contact-rich
    # state, upload that exact fp32 state into the oracle, then compare one
    # substep kernel by kernel -- hash cells, candidate pairs (bit-exact, and
    # non-empty), and every iteration.
    g, gpu, orc = pair(pyoracle, cid, scale)
    gpu.step_frames(frames)
    p4, v4 = gpu.read_f32()
    orc.write_f32(p4, v4)
    orc.write_anchor(gpu.debug_anchor())
    orc.write_rquat(gpu.debug_rquat())
    gpu.debug_prologue()
    orc.integrate()
    orc.candidates()
    assert_same(gpu.debug_keys()[0], orc.keys()[0], "cell hash")
    gcnt, glst = gpu.debug_candidates()
    ocnt, olst = orc.read_candidates()
    assert gcnt.sum() > 0, "expected contacts in this state"
    assert_same(gcnt, ocnt, "candidate counts")
    mask = np.arange(P.NBR_CAP)[None, :] < gcnt[:, None]
    assert_same(np.where(mask, glst, -1), np.where(mask, olst, -1), "candidate lists")
    for it in range(g.cfg.solver_iterations):
        gpu.debug_iteration()
        orc.iteration()
        gp, gv = gpu.read_f32()
        op, ov = orc.read_f32()
        assert_same(gp, op, f"positions after iteration {it}")
        assert_same(gv, ov, f"velocities after iteration {it}")


@pytest.mark.parametrize("cid,scale,frames", [(2, 0, 60), (4, 8, 60)])
def test_near_filter_covers_all_pairs(pbdr, pyoracle, cid, scale, frames):
    # The broadphase filter is exact: every particle with a candidate, and every
    # candidate, is in the filtered (sorted) set.
    g, gpu, orc = pair(pyoracle, cid, scale)
    gpu.step_frames(frames)
    gpu.debug_prologue()
    _, v = gpu.debug_sorted()
    cnt, lst = gpu.debug_candidates()
    near = set(v.tolist())
    mask = np.arange(P.NBR_CAP)[None, :] < cnt[:, None]
    involved = set(np.nonzero(cnt)[0].tolist()) | set(lst[mask].tolist())
    assert involved and involved <= near
    assert len(near) < gpu.n  # the filter actually removes particles


@pytest.mark.slow
@pytest.mark.parametrize("cid", [4, 5])
def test_full_size_properties(pbdr, cid):
    # BASELINE sizes (14.2M / 67.1M particles), where the oracle cannot follow:
    # size-independent properties. (1) Determinism: two handles give
    # bit-identical states. (2) In the first frames no body reaches the ground,
    # so each scene is an isolated system under uniform gravity: its momentum
    # follows P0 - M g t e_z and its angular momentum about its own com is
    # conserved (body-body contacts are equal and opposite, the momentum
    # constraint cancels shape matching's change), to fp32 resolution.
    g = P.GeneratedScene(cid)
    nb = g.desc.num_bodies
    mass = g.array("total_mass", nb)
    scene = g.array("body_scene", nb, np.int64) if cid == 4 else np.zeros(nb, np.int64)
    a = P.GpuSolver(g.desc, g.cfg)
    s0 = a.read_bodies()
    frames = 2
    a.step_frames(frames)
    pa, va = a.read_f32()
    s1 = a.read_bodies()
    b = P.GpuSolver(g.desc, g.cfg)
    b.step_frames(frames)
    pb, vb = b.read_f32()
    assert np.array_equal(pa, pb) and np.array_equal(va, vb)
    assert pa[:, 2].min() > 0.05  # nobody near the ground yet

    def per_scene(st):
        ns = scene.max() + 1
        M = np.bincount(scene, mass, ns)
        C = np.stack([np.bincount(scene, mass * st[:, k], ns) for k in range(3)], 1) / M[:, None]
        Pm = np.stack([np.bincount(scene, st[:, 7 + k], ns) for k in range(3)], 1)
        r = st[:, 0:3] - C[scene]
        Lb = st[:, 10:13] + np.cross(r, st[:, 7:10])
        L = np.stack([np.bincount(scene, Lb[:, k], ns) for k in range(3)], 1)
        return M, Pm, L

    t = frames / g.cfg.frame_rate
    M, P0, L0 = per_scene(s0)
    _, P1, L1 = per_scene(s1)
    expect = P0.copy()
    expect[:, 2] -= M * g.cfg.gravity * t
    assert np.abs(P1 - expect).max() <= 1e-5 * max(1.0, np.abs(expect).max())
    assert np.abs(L1 - L0).max() <= 1e-4 * max(1e-3, np.abs(L0).max())


@pytest.mark.parametrize("coop", ["1", "0"])
def test_one_wave_multi_iteration_path(pbdr, pyoracle, monkeypatch, coop):
    # Scenes whose tiles fit in one wave run a substep's iterations in one
    # cooperative launch (grid barrier per iteration); PBDR_COOP_ITERS=0 forces
    # one launch per iteration. Both equal the oracle bit for bit.
    monkeypatch.setenv("PBDR_COOP_ITERS", coop)
    g = P.GeneratedScene(2)
    gpu = P.GpuSolver(g.desc, g.cfg)
    orc = pyoracle.Oracle(g.desc, g.cfg)
    gpu.step_frames(3)
    assert orc.step(3 * g.cfg.substeps) == 0
    gp, gv = gpu.read_f32()
    op, ov = orc.read_f32()
    assert_same(gp, op, f"coop={coop} positions")
    assert_same(gv, ov, f"coop={coop} velocities")
    assert gpu.info.launches_per_frame > 0


@pytest.mark.parametrize("cluster,kp,fuse", [("1", 0, "1"), ("1", 8, "1"), ("1", 8, "0"), ("0", 8, "1")])
def test_scene_cluster_path(pbdr, pyoracle, monkeypatch, cluster, kp, fuse):
    # Batched scenes (config 4) run a substep's iterations in one launch, one
    # thread-block cluster per scene (its tiles), with a cluster barrier per
    # iteration, and integrate the next substep of the frame in the final
    # writeback; PBDR_CLUSTER_ITERS=0 forces one launch per iteration,
    # PBDR_FUSE_INTEGRATE=0 the separate integrate kernel. All equal the
    # oracle bit for bit through body-body and ground contact.
    monkeypatch.setenv("PBDR_CLUSTER_ITERS", cluster)
    monkeypatch.setenv("PBDR_FUSE_INTEGRATE", fuse)
    g = P.GeneratedScene(4, scale=6)
    g.desc.tile_kp = kp
    gpu = P.GpuSolver(g.desc, g.cfg)
    if cluster == "1":
        # KP = 2 (the small-scene default): 4 warps per cube, 8 tiles per
        # scene; KP = 8: one warp per cube, 2 tiles per scene.
        assert gpu.info.scene_cluster == (2 if kp == 8 else 8)
    else:
        assert gpu.info.scene_cluster == 0
    orc = pyoracle.Oracle(g.desc, g.cfg)
    frames = 100
    gpu.step_frames(frames)
    assert orc.step(frames * g.cfg.substeps) == 0
    gp, gv = gpu.read_f32()
    op, ov = orc.read_f32()
    assert_same(gp, op, f"cluster={cluster} kp={kp} fuse={fuse} positions")
    assert_same(gv, ov, f"cluster={cluster} kp={kp} fuse={fuse} velocities")
    gpu.debug_prologue()
    assert gpu.debug_candidates()[0].sum() > 0, "expected contacts by now"


def test_scene_partners_equal_coarse_grid(pbdr, monkeypatch):
    # Batched scenes find body partners per scene (k_scene_partners) instead of
    # on the coarse body grid, and keep the axis-aligned near test; the coarse
    # path adds the oriented-box test, which may only shrink the near set. The
    # candidate lists are identical in all three set-ups once bodies touch
    # (config 4, after landing).
    out = []
    for scene, obb in (("1", "1"), ("0", "0"), ("0", "1")):
        monkeypatch.setenv("PBDR_SCENE_PARTNERS", scene)
        monkeypatch.setenv("PBDR_OBB", obb)
        g = P.GeneratedScene(4, scale=6)
        gpu = P.GpuSolver(g.desc, g.cfg)
        gpu.step_frames(90)
        gpu.debug_prologue()
        k, v = gpu.debug_sorted()
        cnt, lst = gpu.debug_candidates()
        out.append((np.sort(v), cnt, np.where(np.arange(P.NBR_CAP)[None, :] < cnt[:, None], lst, -1)))
    assert out[0][1].sum() > 0
    assert_same(out[0][0], out[1][0], "near set (axis-aligned test, both partner searches)")
    assert set(out[2][0].tolist()) <= set(out[1][0].tolist())
    for o in out[1:]:
        assert_same(out[0][1], o[1], "candidate counts")
        assert_same(out[0][2], o[2], "candidate lists")


def test_scene_cluster_force_programs(pbdr, pyoracle):
    # Force programs (no torque) on batched scenes keep the fused path: the
    # next substep's integrate inside the cluster launch applies F/M, gravity
    # exemption and the [t_start, t_stop) window (it opens and closes inside
    # the first frame) exactly as the integrate kernel does.
    g = P.GeneratedScene(4, scale=4)
    rng = np.random.default_rng(5)
    progs = []
    for b in range(g.desc.num_bodies):
        kind = b % 4
        F = tuple(rng.uniform(-3, 3, 3)) if kind in (1, 3) else (0.0, 0.0, 0.0)
        t0, t1 = (0.0015, 0.0032) if kind == 3 else (0.0, float("inf"))
        progs.append(P.ForceProgram(F, (0.0, 0.0, 0.0), t0, t1, int(kind == 2), 0))
    sc = P.scene_with_programs(g, progs)
    gpu = P.GpuSolver(sc.desc, g.cfg)
    assert gpu.info.scene_cluster > 0
    orc = pyoracle.Oracle(sc.desc, g.cfg)
    gpu.step_frames(3)
    assert orc.step(3 * g.cfg.substeps) == 0
    gp, gv = gpu.read_f32()
    op, ov = orc.read_f32()
    assert_same(gp, op, "positions")
    assert_same(gv, ov, "velocities")


@pytest.mark.parametrize("cid,scale,frames", [(3, 250, 200), (5, 6, 40)])
def test_isolated_tile_split(pbdr, pyoracle, monkeypatch, cid, scale, frames):
    # Tiles whose bodies have no broadphase partner this substep iterate all of
    # the substep's iterations in one launch (state in shared memory); the
    # others iterate launch by launch. With the one-wave cooperative path off,
    # the split path equals the unsplit one bit for bit through landing and
    # body-body contact, and the oracle over the first frames.
    monkeypatch.setenv("PBDR_COOP_ITERS", "0")
    runs = []
    for split in ("1", "0"):
        monkeypatch.setenv("PBDR_SPLIT_ISOLATED", split)
        g = P.GeneratedScene(cid, scale=scale)
        gpu = P.GpuSolver(g.desc, g.cfg)
        if split == "1":
            orc = pyoracle.Oracle(g.desc, g.cfg)
            gpu.step_frames(2)
            assert orc.step(2 * g.cfg.substeps) == 0
            gp, gv = gpu.read_f32()
            op, ov = orc.read_f32()
            assert_same(gp, op, "split positions vs oracle")
            assert_same(gv, ov, "split velocities vs oracle")
            gpu.step_frames(frames - 2)
        else:
            gpu.step_frames(frames)
        gpu.debug_prologue()
        runs.append((gpu.read_f32(), gpu.debug_candidates()[0].sum()))
    assert runs[0][1] > 0, "expected contacts by the end"
    assert_same(runs[0][0][0], runs[1][0][0], "positions split vs unsplit")
    assert_same(runs[0][0][1], runs[1][0][1], "velocities split vs unsplit")
