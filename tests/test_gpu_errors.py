"""Error behaviour of the GPU path (errors.hpp:8-44 classes through the C-ABI
status codes), cross-checked against the oracle's error record on the same
inputs: degenerate shape matching, candidate overflow and non-finite state."""
import numpy as np
import pytest

from paper_2603_14634_b200 import pbdr as P

pytestmark = pytest.mark.gpu


def _lattice(nx, ny, nz, s=0.02, origin=(0.0, 0.0, 1.0)):
    g = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1).reshape(-1, 3)
    return g * s + np.array(origin)


def test_planar_body_is_degenerate(pbdr, pyoracle):
    # A one-layer body: Apq has rank 2, so the polar of shape matching is
    # degenerate -> DegenerateConfigError (math.cpp:172; P7/polar).
    x = _lattice(5, 5, 1)
    sc = P.ArrayScene(**P.rigid_body_arrays([x], 0.01, [1.0]), has_ground=False)
    cfg = P.solver_cfg()
    gpu = P.GpuSolver(sc.desc, cfg)
    with pytest.raises(P.DegenerateConfigError):
        gpu.step(1)
    o = pyoracle.Oracle(sc.desc, cfg, threads=1)
    assert o.step(1) == P.ERR_DEGENERATE


def test_candidate_overflow_is_reported(pbdr, pyoracle):
    # Twelve interpenetrating bodies: a particle sees more than 32 other-body
    # particles within h -> SimulationError (never a silent truncation, P4).
    rng = np.random.default_rng(2)
    bodies = [_lattice(4, 4, 4, origin=tuple(np.array([0.0, 0.0, 1.0]) + rng.uniform(-0.01, 0.01, 3)))
              for _ in range(12)]
    sc = P.ArrayScene(**P.rigid_body_arrays(bodies, 0.01, [1.0] * 12), has_ground=False)
    cfg = P.solver_cfg()
    gpu = P.GpuSolver(sc.desc, cfg)
    with pytest.raises(P.SimulationError):
        gpu.step(1)
    o = pyoracle.Oracle(sc.desc, cfg, threads=1)
    assert o.step(1) == P.ERR_SIMULATION
    assert o.error()[1] & 4  # PBDR_DEVERR_NBR_OVERFLOW


def test_non_finite_state_is_reported(pbdr):
    # A NaN velocity propagates into the body sums -> SimulationError with the
    # frame index in the payload (errors.hpp:39-44).
    g = P.GeneratedScene(2)
    gpu = P.GpuSolver(g.desc, g.cfg)
    gpu.step_frames(1)
    p4, v4 = gpu.read_f32()
    v4[5, 0] = np.nan
    gpu.write_f32(None, v4)
    with pytest.raises(P.SimulationError) as e:
        gpu.step_frames(1)
    assert "non-finite" in str(e.value)


def test_oversized_body_is_a_config_error(pbdr):
    # Bodies above one CTA run on a cluster of up to 16 CTAs (32768
    # particles, tests/test_gpu_big_bodies.py); beyond that: ConfigError.
    x = _lattice(33, 33, 31)  # 33759 > 32768 particles
    sc = P.ArrayScene(**P.rigid_body_arrays([x], 0.01, [1.0]), has_ground=False)
    with pytest.raises(P.ConfigError):
        P.GpuSolver(sc.desc, P.solver_cfg())
