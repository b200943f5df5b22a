"""dist.py's default CudaOps path on one GPU (NCCL process group of size 1):
Mode A and Mode B through the library kernels, checked against the oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import datagen
import oracle
from paper_2605_10390_b200 import dist as fsdist

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group(cuda):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda)
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["B", "A"])
@pytest.mark.parametrize("dist_name", ["uniform", "zipf", "const"])
def test_dist_single_rank(cuda, nccl_group, mode, dist_name):
    keys = datagen.gen_u16(dist_name, 1_000_003, seed=1)
    out, (b, e) = fsdist.sort_keys_u16(torch.from_numpy(keys).to(cuda), mode=mode)
    assert (b, e) == (0, keys.size)
    np.testing.assert_array_equal(out.cpu().numpy(), oracle.sort_u16(keys))
