"""Per-rank device memory of the 8-GPU cfg5 run (BASELINE cfg5: t = 4e6 rows
sharded over 8 GPUs, n = 96, b = 6, C2..C6): one rank's shard (t = 500,000
rows of the recipe) through the sample-split path (distributed.py, NCCL,
world size 1 on this 1-GPU pool) -- the packed tensors dominate (M_6 alone is
2.53e9 doubles = 20.25 GB), so this is the footprint every rank of the 8-GPU
run needs.  Target <= 25 GB; the peak is printed."""

import json
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

LIMIT_GB = 25.0


def _worker(rank, port, out):
    import torch.distributed as dist

    import workloads
    from paper_1701_05420_b200.distributed import cumulants_upto_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    x = torch.from_numpy(workloads.generate("cfg5", 500_000)).cuda()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    mean, ts = cumulants_upto_sharded(x, 6, 6)
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated()
    c6 = ts[-1]
    rec = {"peak_gb": peak / 1e9, "input_gb": base / 1e9, "c6_elements": int(c6.numel()),
           "c6_finite": bool(torch.isfinite(c6).all().item())}
    with open(out, "w") as f:
        json.dump(rec, f)
    dist.destroy_process_group()


def test_cfg5_rank_shard_peak_memory(tmp_path):
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "mem.json")
    mp.spawn(_worker, args=(port, out), nprocs=1, join=True)
    rec = json.load(open(out))
    print(f"cfg5 rank shard (t=500000, n=96, b=6, C2..C6): peak device memory {rec['peak_gb']:.2f} GB "
          f"(input {rec['input_gb']:.2f} GB)")
    path = os.environ.get("BCG_HIGHORDER_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"test": "cfg5_rank_shard_memory", **rec}) + "\n")
    assert rec["c6_finite"] and rec["c6_elements"] == 2_531_741_184
    assert rec["peak_gb"] <= LIMIT_GB
