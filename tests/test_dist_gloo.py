"""Multi-process (world_size 2, gloo, CPU) tests of the data-parallel driver:
shard arithmetic, template broadcast, and result gather order -- the N>1 host
logic bench.py runs over NCCL.  The per-rank aligner here is the CPU oracle
(test infrastructure), so no GPU is needed; the gathered trajectory must equal
the unsharded oracle run frame for frame."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1506_06039_b200.dist import align_sharded, broadcast_template, shard_range


def test_shard_range_partitions():
    for T in [0, 1, 7, 20, 10000, 50001]:
        for world in [1, 2, 3, 8]:
            spans = [shard_range(T, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == T
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
            per = (T + world - 1) // world
            assert all(b - a <= per for a, b in spans)
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, T, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from synth import config_spec, make_stack
        spec = config_spec(1, m=48, n=48, w=6, T=T, n_blobs=12, shift_bound=4)
        if rank == 0:
            tpl = make_stack(spec, 0, 1).template.clone()
        else:
            tpl = torch.zeros((48, 48), dtype=torch.int32).to(torch.uint16)
        broadcast_template(tpl)
        lo, hi = shard_range(T, world, rank)
        local = make_stack(spec, lo, hi - lo).frames if hi > lo else torch.zeros((0, 48, 48), dtype=torch.uint16)

        def align_fn(fr):
            sh, fm = oracle.align_stack(fr.numpy(), tpl.numpy(), spec.w, spec.levels, workers=1)
            return torch.from_numpy(sh), torch.from_numpy(fm), None

        sh, fm, _ = align_sharded(local, T, align_fn)
        if rank == 0:
            q.put((sh.numpy().tolist(), fm.numpy().tolist(), tpl.numpy().tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("T", [7, 10])
def test_gloo_world2_gather_equals_unsharded(T):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, T, q)) for r in range(2)]
    for p in ps:
        p.start()
    import queue
    import time
    t0 = time.time()
    while True:
        try:
            sh, fm, tpl = q.get(timeout=2)
            break
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in ps) or time.time() - t0 > 240:
                for p in ps:
                    p.kill()
                raise AssertionError("a gloo worker failed")
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle
    from synth import config_spec, make_stack
    spec = config_spec(1, m=48, n=48, w=6, T=T, n_blobs=12, shift_bound=4)
    st = make_stack(spec, 0, T)
    assert np.array_equal(np.array(tpl, np.uint16), st.template.numpy())
    ref_sh, ref_fm = oracle.align_stack(st.frames.numpy(), st.template.numpy(), spec.w, spec.levels)
    assert np.array_equal(np.array(sh), ref_sh)
    assert np.array_equal(np.array(fm), ref_fm)
