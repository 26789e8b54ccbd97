"""Multi-rank host logic on CPU (gloo, world_size 2): sequence sharding, the
max-over-ranks clock and the final pose gather used by bench.py --gpus N.
Each rank builds its own sequence's window (graph + flattening, host C++)
and the gathered poses must equal what each rank would compute alone."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2208_04726_b200.dist import shard


def test_shard_partitions_contiguously():
    for n in (1, 7, 1024):
        for w in (1, 2, 4, 8):
            got = [list(shard(n, r, w)) for r in range(w)]
            assert sum(got, []) == list(range(n))
            sizes = [len(g) for g in got]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2208_04726_b200 import PatchGraph

    import pvo_synth as synth
    from paper_2208_04726_b200.dist import gather_poses, max_over_ranks, shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        seqs = list(shard(4, rank, world))
        flat = []
        for s in seqs:
            w = synth.generate("c1", seed=100 + s, features=False, frames=6, patches=8)
            prob = synth.build_graph(w, PatchGraph).window_problem(w.cfg["window"])
            flat.append(prob["poses"])
        poses = np.concatenate(flat)
        t = max_over_ranks([float(rank + 1), float(len(seqs))])
        gathered = gather_poses(poses)
        q.put((rank, seqs, t.tolist(), [g.tolist() for g in gathered]))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_shard_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, s0, t0, g0), (r1, s1, t1, g1) = res
    assert s0 == [0, 1] and s1 == [2, 3]
    assert t0 == t1 == [2.0, 2.0]  # MAX over ranks
    assert g0 == g1  # every rank sees the same gathered list
    # the gathered block of each rank equals an independent single-process run
    from paper_2208_04726_b200 import PatchGraph
    import pvo_synth as synth

    for rank, seqs in ((0, s0), (1, s1)):
        ref = []
        for s in seqs:
            w = synth.generate("c1", seed=100 + s, features=False, frames=6, patches=8)
            ref.append(synth.build_graph(w, PatchGraph).window_problem(w.cfg["window"])["poses"])
        assert np.array_equal(np.asarray(g0[rank]), np.concatenate(ref))
