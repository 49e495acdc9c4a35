"""The sharded (multi-GPU) path through NCCL at world size 1 on one B200:
CUDA powersort of the shard, splitters, all-to-all-v, CUDA stable merge."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_sharded_sort_world1_nccl():
    import torch
    import torch.distributed as dist

    from paper_1805_04154_b200 import dist as rsd
    from paper_1805_04154_b200 import workloads

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl")
    try:
        k, t = workloads.config4(200000, seed=3, mean=100.0)
        keys = torch.from_numpy(k.copy()).cuda()
        tags = torch.from_numpy(t.copy()).cuda()
        out, tout, info = rsd.sharded_sort(keys, tags)
        order = np.argsort(k, kind="stable")
        assert np.array_equal(out.cpu().numpy(), k[order])
        assert np.array_equal(tout.cpu().numpy(), t[order])
    finally:
        dist.destroy_process_group()
