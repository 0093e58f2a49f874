"""X-slab decomposition of one scene (config 5).

CPU: the runner drives the oracle on gloo ranks (world 2, spawned processes)
and on in-process thread ranks (world 3, LocalComm); the union of the ranks'
owned bodies after several frames -- including repartitions and migrations
across a slab boundary -- equals the single-process run bit for bit.
GPU: the same runner over the C-ABI (set_roles / gather / scatter / staged
stepping), ranks as threads on one device, against one whole-scene handle.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2603_14634_b200 import pbdr as P
from paper_2603_14634_b200 import slab as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GX = 8        # config-5 grid 8 x 8 x 4 = 256 cubes of 512 particles
FRAMES = 3
MARGIN = 0.05


class _Scene:
    """Config 5 at 8 x 8 x 4 cubes with x-velocities +-1.5 m/s by grid column
    (odd columns +x, even -x), so column pairs collide within a few frames --
    also across the slab edges the tests place. `torque`: every body also
    carries a torque program (ghosts then need exact anchors for the wrench)."""

    def __init__(self, fast=False, torque=False):
        g = P.GeneratedScene(5, seed=0, scale=GX)
        self.cfg = g.cfg
        nb = g.desc.num_bodies
        off = g.array("body_offsets", nb + 1, np.int64)
        rng = np.random.default_rng(5)
        progs = [P.ForceProgram((0, 0, 0), tuple(rng.uniform(-0.02, 0.02, 3)) if torque else (0, 0, 0), 0.0,
                                float("inf"), 0, 0) for _ in range(nb)]
        self.sc = P.scene_with_programs(g, progs)
        com_x = self.sc.rest_com[:, 0]
        col = np.rint((com_x - com_x.min()) / 0.2).astype(int)
        body = np.repeat(np.arange(nb), np.diff(off))
        vx = np.where(col % 2 == 1, 1.5, -1.5)
        self.sc.velocity[self.sc.body_indices, 0] += vx[body]
        if fast:
            self.sc.velocity[:, 0] += 10.0  # 42 mm per frame: beyond margin / 2
        self.desc, self.off, self.nb = self.sc.desc, off, nb
        self.rho, self.h = S.body_reach(self.sc.rest_offsets, off, self.sc.radius)


def _scene(fast=False, torque=False):
    sc = _Scene(fast, torque)
    return sc, sc.off, sc.rho, sc.h


def _crossing_geometry(world, com_frames, rho, h):
    """Slab edges where column pairs collide (odd column moving +x meets the
    next even column moving -x), each at the median final com of the left
    column's bodies: bodies on both sides are in contact across the edge and
    left-column bodies that started below the edge migrate during the run."""
    c0, c1 = com_frames[0], com_frames[-1]
    col = np.rint((c0 - c0.min()) / 0.2).astype(int)
    mids = sorted({k for k in col.tolist() if k % 2 == 1 and k + 1 <= col.max()})  # left column of each pair
    pick = {2: [mids[len(mids) // 2]], 3: [mids[0], mids[-1]]}[world]
    edges = [-np.inf] + [float(np.median(c1[col == k])) for k in pick] + [np.inf]
    return S.SlabGeometry(np.array(edges), 2.0 * rho + h + MARGIN, MARGIN)


def _reference(pyoracle, g):
    o = pyoracle.Oracle(g.desc, g.cfg)
    coms = [o.body_stats()[:, 0].copy()]
    for _ in range(FRAMES):
        assert o.step(g.cfg.substeps) == 0
        coms.append(o.body_stats()[:, 0].copy())
    p4, v4 = o.read_f32()
    # inter-body contact candidates at the end of the run (the halo has work)
    o.integrate()
    o.candidates()
    cnt, lst = o.read_candidates()
    body = np.repeat(np.arange(g.nb), np.diff(g.off))
    ii = np.repeat(np.arange(len(cnt)), cnt)
    jj = lst[np.arange(P.NBR_CAP)[None, :] < cnt[:, None]]
    return p4, v4, coms, (body[ii], body[jj])


def _cross_pairs(pairs, com, geo):
    bi, bj = pairs
    s = geo.slab_of(com)
    return int(np.count_nonzero(s[bi] != s[bj]))


def _check_union(states, p_ref, v_ref, nb):
    owned = np.concatenate([s[0] for s in states])
    assert np.array_equal(np.sort(owned), np.arange(nb)), "every body owned by exactly one rank"
    for ids, slots, p4, v4 in states:
        assert np.array_equal(p4, p_ref[slots]), "owned positions differ from the single-process run"
        assert np.array_equal(v4, v_ref[slots]), "owned velocities differ from the single-process run"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, out_dir, edges, band):
    for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
        sys.path.insert(0, p)
    import torch.distributed as dist
    import pyoracle
    from slab_oracle_engine import OracleEngine
    from paper_2603_14634_b200 import slab as S2

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, off, _, _ = _scene()
    eng = OracleEngine(pyoracle.Oracle(g.desc, g.cfg, threads=2), g.cfg)
    geo = S2.SlabGeometry(np.array(edges), band, MARGIN)
    run = S2.SlabRunner(eng, rank, world, S2.TorchComm(), off, geometry=geo)
    run.start()
    run.step_frames(FRAMES)
    ids, slots, p4, v4 = run.owned_state()
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), ids=ids, slots=slots, p4=p4, v4=v4,
             migrations=run.migrations)
    dist.barrier()
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def reference(pyoracle):
    g, off, rho, h = _scene()
    p4, v4, coms, pairs = _reference(pyoracle, g)
    return g, off, rho, h, p4, v4, coms, pairs


def test_slab_gloo_world2_matches_single_process(reference, tmp_path):
    g, off, rho, h, p_ref, v_ref, coms, pairs = reference
    geo = _crossing_geometry(2, coms, rho, h)
    assert _cross_pairs(pairs, coms[-1], geo) > 0, "contacts across the slab edge"
    mp.start_processes(_gloo_worker, args=(2, _free_port(), str(tmp_path), geo.edges.tolist(), geo.ghost_band),
                       nprocs=2, join=True, start_method="spawn")
    states, migr = [], 0
    for r in range(2):
        z = np.load(tmp_path / f"r{r}.npz")
        states.append((z["ids"], z["slots"], z["p4"], z["v4"]))
        migr += int(z["migrations"])
    _check_union(states, p_ref, v_ref, g.nb)
    assert migr >= 1, "the edge placement should move at least one body across"


def test_slab_threads_world3_matches_single_process(reference, pyoracle):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from slab_oracle_engine import OracleEngine
    g, off, rho, h, p_ref, v_ref, coms, pairs = reference
    geo = _crossing_geometry(3, coms, rho, h)
    assert _cross_pairs(pairs, coms[-1], geo) > 0, "contacts across the slab edges"
    engines = [OracleEngine(pyoracle.Oracle(g.desc, g.cfg, threads=2), g.cfg) for _ in range(3)]
    states = S.run_threads(engines, off, FRAMES, geometry=geo)
    _check_union(states, p_ref, v_ref, g.nb)


def test_slab_threads_with_torque_programs(pyoracle):
    # Ghosts integrate locally; with torque programs their wrench prepass uses
    # anchored sums, so the anchors must travel with the halo (substep end).
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from slab_oracle_engine import OracleEngine
    g, off, rho, h = _scene(torque=True)
    p_ref, v_ref, coms, pairs = _reference(pyoracle, g)
    geo = _crossing_geometry(2, coms, rho, h)
    engines = [OracleEngine(pyoracle.Oracle(g.desc, g.cfg, threads=4), g.cfg) for _ in range(2)]
    states = S.run_threads(engines, off, FRAMES, geometry=geo)
    _check_union(states, p_ref, v_ref, g.nb)


def test_slab_geometry_rules():
    geo = S.slab_geometry(np.linspace(-6.3, 6.3, 64), 8, rho=0.1273, h=0.02, margin=0.1)
    assert geo.world == 8 and np.isinf(geo.edges[0]) and np.isinf(geo.edges[-1])
    assert list(geo.slab_of([-7.0, -6.3, 0.0, 6.3, 9.0])) == [0, 0, 4, 7, 7]
    with pytest.raises(P.ConfigError):
        S.slab_geometry(np.linspace(-1, 1, 10), 8, rho=0.1273, h=0.02, margin=0.1)


def test_slab_guard_raises_on_fast_bodies(pyoracle):
    # A body moving faster than margin/2 per frame breaks the ghost-band
    # guarantee: the runner must refuse loudly instead of diverging silently.
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from slab_oracle_engine import OracleEngine
    g, off, rho, h = _scene(fast=True)
    engines = [OracleEngine(pyoracle.Oracle(g.desc, g.cfg, threads=2), g.cfg) for _ in range(2)]
    with pytest.raises(P.SimulationError):
        S.run_threads(engines, off, 2, rho=rho, h=h, margin=MARGIN)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_slab_gpu_threads_bit_exact(pbdr, pyoracle, world):
    g, off, rho, h = _scene()
    whole = P.GpuSolver(g.desc, g.cfg)
    coms = [whole.read_bodies()[:, 0].copy()]
    for _ in range(FRAMES):
        whole.step_frames(1)
        coms.append(whole.read_bodies()[:, 0].copy())
    p_ref, v_ref = whole.read_f32()
    geo = _crossing_geometry(world, coms, rho, h)
    engines = [S.GpuEngine(P.GpuSolver(g.desc, g.cfg), g.cfg) for _ in range(world)]
    states = S.run_threads(engines, off, FRAMES, geometry=geo)
    _check_union(states, p_ref, v_ref, g.nb)
    # and the oracle agrees with the whole-scene GPU run (same pinned semantics)
    o = pyoracle.Oracle(g.desc, g.cfg)
    assert o.step(FRAMES * g.cfg.substeps) == 0
    assert np.array_equal(o.read_f32()[0], p_ref)
