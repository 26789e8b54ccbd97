"""Sequence sharding on the device path: G processes, each owning
a contiguous block of independent sequences (paper_2208_04726_b200.dist.shard),
run the batched corr + BA launches on their block with no communication, then
one gather of the final poses.  Every sequence's result must be bit-identical
for G = 1, 2 and 4, i.e. independent of which sequences share a launch.

The box has one GPU, so the G ranks share cuda:0 and gather over gloo (NCCL
refuses two ranks on one device); the device work per rank is exactly the
bench's (pvo.Batch), only the transport of the final gather differs.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
N_SEQ = 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sequence(sid, ctx, slot0):
    """Window of sequence `sid`: c2-shaped geometry seeded by sid, frame
    features generated on the device from a generator seeded by sid."""
    import torch

    import paper_2208_04726_b200 as pvo
    import pvo_synth as synth

    w = synth.generate("c2", seed=9000 + sid, features=False, frames=12, patches=32)
    g = synth.build_graph(w, pvo.PatchGraph)
    prob = synth.window_arrays(w, g.window_problem(w.cfg["window"]))
    pf = np.random.default_rng(sid).standard_normal((len(prob["depth"]), 2, 9, 128)).astype(np.float32)
    pf /= np.linalg.norm(pf, axis=-1, keepdims=True)
    F = w.cfg["frames"]
    H0, W0 = w.image[1] // 4, w.image[0] // 4
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1000 + sid)
    l0 = torch.randn((F, H0, W0, 128), device="cuda", generator=gen)
    l0 /= l0.norm(dim=-1, keepdim=True)
    l1 = l0.view(F, H0 // 4, 4, W0 // 4, 4, 128).mean(dim=(2, 4))
    l1 = (l1 / l1.norm(dim=-1, keepdim=True).clamp_min(1e-12)).contiguous()
    torch.cuda.synchronize()  # device uploads are ordered on the context's stream, not torch's
    for f in range(F):
        ctx.frames_upload(slot0 + f, l0[f], l1[f], device=True)
    torch.cuda.synchronize()
    return w, prob, pf


def _run_block(seqs):
    import torch

    import paper_2208_04726_b200 as pvo

    ctx = pvo.Context(0)
    try:
        F, H0, W0 = 12, 120, 160
        ctx.frames_reserve(len(seqs) * F, W0, H0, W0 // 4, H0 // 4, 128)
        probs, slots, feats, K, image = [], [], [], None, None
        for i, sid in enumerate(seqs):
            w, prob, pf = _sequence(sid, ctx, i * F)
            probs.append(prob)
            slots.append(prob["pose_frames"] + i * F)
            feats.append(pf)
            K, image = w.K, w.image
        bat = pvo.Batch(ctx)
        bat.load(probs, slots, feats, K, image)
        # NaN-filled: an output the kernels never write would show up (and differ between processes)
        vol = torch.full((bat.n_edges, 2, 9, 7, 7), float("nan"), dtype=torch.float32, device="cuda")
        bat.iteration(2, corr_device_ptr=vol.data_ptr())
        res = bat.read()
        vols = [vol[bat.edge_off[i]:bat.edge_off[i + 1]].cpu().numpy() for i in range(len(seqs))]
        assert not any(np.isnan(v).any() for v in vols), "unwritten correlation outputs"
        return [(r[0], r[1], np.asarray(r[2]), v) for r, v in zip(res, vols)]
    finally:
        ctx.close()


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2208_04726_b200.dist import gather_poses, shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        seqs = list(shard(N_SEQ, rank, world))
        out = _run_block(seqs)
        gathered = gather_poses(np.concatenate([o[0] for o in out]))  # the bench's final collective
        q.put((rank, seqs, [(p.tolist(), d.tolist(), n.tolist(), v.tobytes()) for p, d, n, v in out],
               [g.tolist() for g in gathered]))
    finally:
        dist.destroy_process_group()


def _sharded(world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in procs), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    per_seq = {}
    for rank, seqs, outs, gathered in res:
        assert np.array_equal(np.asarray(gathered[rank]), np.concatenate([np.asarray(o[0]) for o in outs]))
        for sid, o in zip(seqs, outs):
            per_seq[sid] = o
    return per_seq


def test_sequence_results_bit_identical_across_shardings():
    ref = _sharded(1)
    assert sorted(ref) == list(range(N_SEQ))
    for world in (2, 4):
        got = _sharded(world)
        assert sorted(got) == list(range(N_SEQ))
        for sid in range(N_SEQ):
            for name, a, b in zip(("poses", "depths", "norms", "volume"), got[sid], ref[sid]):
                assert a == b, (world, sid, name)
