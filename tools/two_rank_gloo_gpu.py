"""Two ranks on ONE GPU over gloo (host-staged collectives, so no rank's
kernel waits on another's): the real CUDA per-rank path of both multi-GPU
modes at world size 2, against the single-process result.

    python tools/two_rank_gloo_gpu.py
"""
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def worker(rank, world, port, x, m, b, out):
    from paper_1701_05420_b200.distributed import cumulants_upto_block_split, cumulants_upto_sharded, shard_bounds

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_bounds(x.shape[0], world, rank)
    mean, ts = cumulants_upto_sharded(torch.from_numpy(x[lo:hi]).cuda(), m, b)
    mean2, ts2 = cumulants_upto_block_split(torch.from_numpy(x).cuda(), m, b)
    np.savez(f"{out}_{rank}.npz", mean=mean.cpu().numpy(), mean2=mean2.cpu().numpy(),
             **{f"c{k}": t.cpu().numpy() for k, t in enumerate(ts, 2)},
             **{f"d{k}": t.cpu().numpy() for k, t in enumerate(ts2, 2)})
    dist.destroy_process_group()


def main():
    import paper_1701_05420_b200 as bcg

    rng = np.random.default_rng(5)
    for (t, n, m, b) in [(5001, 9, 6, 3), (4000, 12, 5, 4), (3000, 16, 4, 8)]:
        x = rng.exponential(1.0, (t, n)) + rng.standard_normal((t, n))
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        out = f"/tmp/two_rank_{t}"
        mp.spawn(worker, args=(2, port, x, m, b, out), nprocs=2, join=True)
        cs = bcg.cumulants_upto(x, m, b=b)
        worst = 0.0
        for r in range(2):
            got = np.load(f"{out}_{r}.npz")
            np.testing.assert_allclose(got["mean"], cs[1], rtol=1e-13)
            for k in range(2, m + 1):
                want = cs[k].packed_host()
                np.testing.assert_allclose(got[f"c{k}"], want, rtol=1e-9, atol=1e-12)
                np.testing.assert_array_equal(got[f"d{k}"], want)  # block split: bitwise
                worst = max(worst, float(np.max(np.abs(got[f"c{k}"] - want) / np.maximum(np.abs(want), 1e-3))))
        print(f"t={t} n={n} m={m} b={b}: both ranks match (sample split max rel dev {worst:.1e}; block split bitwise)",
              flush=True)


if __name__ == "__main__":
    main()
