"""The view-sharded training path on one GPU: a 1-rank NCCL group with the
union gradient exchange forced on must train like the local path (same
counters; parameters equal up to the f32 wire rounding of the gradients)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu

from paper_2507_01110_b200.core import SECTIONS, AttributeArrays  # noqa: E402

from .test_train_gpu import make_case  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_union_allreduce_path_matches_local():
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        a, _, lrs = make_case()
        b, _, _ = make_case()
        b.distributed = True
        for it in range(1, 6):
            ra, rb = a.train_step(it), b.train_step(it)
            for k in ("view", "gaussians_rendered", "gaussians_loaded_from_store", "cache_hits",
                      "bytes_streamed"):
                assert ra[k] == rb[k], (it, k)
            assert abs(ra["loss"] - rb["loss"]) <= 1e-4 * abs(ra["loss"])
        assert b._last_union[0].numel() == ra["gaussians_rendered"]
        pa = AttributeArrays.from_packed(a.scene.params.cpu().numpy(), a.scene.cap)
        pb = AttributeArrays.from_packed(b.scene.params.cpu().numpy(), b.scene.cap)
        for name, _ in SECTIONS:
            x, y = getattr(pa, name), getattr(pb, name)
            lr = lrs[name] if name not in ("scales", "opacities") else 1.0
            assert np.all(np.abs(x - y) <= 5 * 2.5 * lr * np.maximum(1.0, np.abs(x)) + 1e-12), name
            assert np.mean(np.abs(x - y) <= 1e-5 * np.maximum(1.0, np.abs(x))) > 0.98, name
        assert torch.equal(a.scene.step, b.scene.step)
    finally:
        dist.destroy_process_group()
