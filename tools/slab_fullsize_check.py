"""Full-size config-5 x-slab check on one GPU: two thread ranks (LocalComm,
one handle each on the same device) against one whole-scene handle, 2 frames,
owned states compared bit for bit. Not a scaling measurement."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_14634_b200 import pbdr as P  # noqa: E402
from paper_2603_14634_b200 import slab as S  # noqa: E402

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 2
world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
g = P.GeneratedScene(5)
nb = g.desc.num_bodies
off = g.array("body_offsets", nb + 1, np.int64)
rho, h = S.body_reach(g.array("rest_offsets", 3 * g.num_particles), off, g.array("radius", g.num_particles))
whole = P.GpuSolver(g.desc, g.cfg)
whole.step_frames(frames)
p_ref, v_ref = whole.read_f32()
whole.close()
engines = [S.GpuEngine(P.GpuSolver(g.desc, g.cfg), g.cfg) for _ in range(world)]
t0 = time.perf_counter()
states = S.run_threads(engines, off, frames, rho=rho, h=h, margin=0.1)
dt = time.perf_counter() - t0
owned = np.concatenate([s[0] for s in states])
assert np.array_equal(np.sort(owned), np.arange(nb))
ok = all(np.array_equal(p4, p_ref[slots]) and np.array_equal(v4, v_ref[slots]) for _, slots, p4, v4 in states)
print(f"C5 full size, {world} thread ranks, {frames} frames: owned states bit-identical to one handle: {ok}; "
      f"ghost-free owned counts {[len(s[0]) for s in states]}; wall {dt:.1f} s")
assert ok
