"""Multi-rank (world_size 2, gloo, CPU) tests of the config-4 scene sharding:
each rank generates and simulates its own scene range with the CPU oracle; the
union of the rank results equals the single-process run bit for bit (scenes
are independent, so the data path needs no collective), and the timing /
aggregate reductions behave as bench.py uses them."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCENES_PER_RANK = 3
SUBSTEPS = 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    for p in (ROOT, os.path.join(ROOT, "oracle")):
        sys.path.insert(0, p)
    import torch.distributed as dist
    from paper_2603_14634_b200 import shard as S
    import pyoracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sh = S.c4_shard(rank, world, SCENES_PER_RANK)
    g = S.generate_c4_shard(sh, seed=0)
    o = pyoracle.Oracle(g.desc, g.cfg, threads=2)
    assert o.step(SUBSTEPS) == 0
    p4, v4 = o.read_f32()
    np.save(os.path.join(out_dir, f"pos_{rank}.npy"), p4)
    np.save(os.path.join(out_dir, f"vel_{rank}.npy"), v4)
    # bench.py's reductions: max of device time, sum of aggregates.
    t = S.max_over_ranks(float(rank + 1))
    m = 1.0 / g.array("inv_mass", g.num_particles)
    agg = S.sum_over_ranks([g.num_particles, float((m[:, None] * v4[:, :3]).sum())])
    np.save(os.path.join(out_dir, f"red_{rank}.npy"), np.array([t, agg[0], agg[1]]))
    dist.barrier()
    dist.destroy_process_group()


def test_c4_shards_match_single_process(tmp_path, pbdr, pyoracle):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    from paper_2603_14634_b200 import shard as S
    whole = S.generate_c4_shard(S.c4_shard(0, 1, world * SCENES_PER_RANK))
    o = pyoracle.Oracle(whole.desc, whole.cfg, threads=2)
    assert o.step(SUBSTEPS) == 0
    p4, v4 = o.read_f32()
    cat_p = np.concatenate([np.load(tmp_path / f"pos_{r}.npy") for r in range(world)])
    cat_v = np.concatenate([np.load(tmp_path / f"vel_{r}.npy") for r in range(world)])
    assert np.array_equal(cat_p, p4) and np.array_equal(cat_v, v4)
    reds = [np.load(tmp_path / f"red_{r}.npy") for r in range(world)]
    assert all(r[0] == float(world) for r in reds)  # max over ranks
    assert all(r[1] == whole.num_particles for r in reds)  # sum over ranks
    m = 1.0 / whole.array("inv_mass", whole.num_particles)
    np.testing.assert_allclose(reds[0][2], (m[:, None] * v4[:, :3]).sum(), rtol=1e-9)


def test_shard_ranges():
    from paper_2603_14634_b200 import shard as S
    sh = S.c4_shard(3, 8, 4096)
    assert sh.first_scene == 3 * 4096 and sh.total_scenes == 8 * 4096
    assert list(S.c4_shard(1, 2, 3).scenes) == [3, 4, 5]
    with pytest.raises(ValueError):
        S.c4_shard(2, 2)
