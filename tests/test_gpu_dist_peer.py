"""Fused results gather over peer memory (dist.PeerResults): the
library's kernels write each frame's record through views of rank 0's symmetric-memory
buffers.  One GPU here (world size 1, NCCL): the records must be bit-identical to an
align into ordinary device buffers, and visible in rank 0's buffer after the barrier."""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_peer_results_world1():
    import torch.distributed as dist
    from paper_1506_06039_b200 import Plan
    from paper_1506_06039_b200.dist import PeerResults
    from synth import config_spec, make_stack
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        T = 1300                                        # > one internal batch: pipelined TC path
        spec = config_spec(2, T=T)
        st = make_stack(spec, 0, T, device=dev)
        p = Plan(spec.m, spec.n, spec.w, spec.levels, spec.dtype, 12, device=0)
        p.set_template(st.template)
        sh = torch.empty((T, 2), dtype=torch.int32, device=dev)
        fm = torch.empty((T,), dtype=torch.float64, device=dev)
        co = torch.empty_like(st.frames)
        p.align_into(st.frames, sh, fm, co)
        pr = PeerResults(T, dev)
        pr.shifts.fill_(-7)
        pr.fmin.fill_(-1.0)
        p.align_into(st.frames, pr.shifts, pr.fmin, co)
        pr.barrier()
        torch.cuda.synchronize()
        gs, gf = pr.gathered(T)
        assert torch.equal(gs, sh) and torch.equal(gf.view(torch.int64), fm.view(torch.int64))
    finally:
        dist.destroy_process_group()
