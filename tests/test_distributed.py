"""Multi-process (gloo, world size 2 and 3) tests of the multi-GPU paths'
collective logic (distributed.py): the sample split (all-reduce of the lower
orders, reduce-scatter + all-gather of the top two) and the block split.  The per-rank kernels are replaced by the
CPU oracle, so this runs on a GPU-less host; the CUDA ops are covered by the
GPU parity tests."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc
from paper_1701_05420_b200.distributed import (
    block_bounds,
    cumulants_upto_block_split,
    cumulants_upto_sharded,
    shard_bounds,
)
from paper_1701_05420_b200.layout import layout


class OracleOps:
    """Per-rank compute on the CPU oracle (test stand-in for CudaOps)."""

    def matrix(self, x):
        return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64))

    def colstats(self, X):
        a = X.numpy()
        bad = np.argwhere(~np.isfinite(a))
        first = int(bad[0][0] * a.shape[1] + bad[0][1]) if len(bad) else -1
        return torch.as_tensor(a.sum(0)), torch.as_tensor((a * a).sum(0)), torch.tensor([first])

    def colmean(self, X):
        s, _, bad = self.colstats(X)
        return s / X.shape[0], bad

    def center(self, X, mean):
        return X - mean

    def centered_stats(self, Xc):
        s, q, _ = self.colstats(Xc)
        return s, q

    def moment_raw(self, X, k, b, key_range=None, size=None):
        full = torch.as_tensor(orc.moment_raw_sums(X.numpy(), k, b))
        out = torch.zeros(max(full.numel(), size or 0), dtype=full.dtype)
        if key_range is None:
            out[:full.numel()] = full
            return out
        lay = layout(X.shape[1], k, b)
        lo, hi = int(lay.offs[key_range[0]]), int(lay.offs[key_range[1]])
        out[lo:hi] = full[lo:hi]
        return out

    def divide(self, buf, t):
        buf /= t

    def recursion_span(self, mk, n, k, b, lower, e0, e1, central=None):
        # element-wise: the elements outside [e0, e1) hold unreduced sums on
        # this rank, but no element of the span reads them
        S = layout(n, k, b).size
        full = orc.cumulant_from_moment(mk[:S].numpy().copy(), k, {j: v.numpy() for j, v in lower.items()}, n, b)
        mk[e0:e1] = torch.as_tensor(full[e0:e1])

    def recursion_range(self, mk, n, k, b, lower, k0, k1, central=None):
        full = orc.cumulant_from_moment(mk.numpy().copy(), k, {j: v.numpy() for j, v in lower.items()}, n, b)
        lay = layout(n, k, b)
        lo, hi = int(lay.offs[k0]), int(lay.offs[k1])
        mk[lo:hi] = torch.as_tensor(full[lo:hi])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, x, m_max, b, out_path, mode="samples"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if mode == "samples":
        lo, hi = shard_bounds(x.shape[0], world, rank)
        mean, tensors = cumulants_upto_sharded(x[lo:hi], m_max, b, ops=OracleOps())
    else:
        mean, tensors = cumulants_upto_block_split(x, m_max, b, ops=OracleOps())
    np.savez(f"{out_path}_{rank}.npz", mean=mean.numpy(), **{f"c{k}": t.numpy() for k, t in enumerate(tensors, 2)})
    dist.destroy_process_group()


def test_shard_and_block_bounds():
    assert [shard_bounds(101, 4, r) for r in range(4)] == [(0, 25), (25, 50), (50, 75), (75, 101)]
    spans = [block_bounds(330, 8, r) for r in range(8)]
    assert spans[0][0] == 0 and spans[-1][1] == 330
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


@pytest.mark.parametrize("world,mode,m_max,b", [(2, "samples", 6, 2), (3, "samples", 5, 3), (2, "blocks", 6, 2),
                                                (3, "blocks", 6, 3), (4, "samples", 6, 3), (3, "samples", 4, 2)])
def test_sharded_cumulants_match_oracle(world, mode, m_max, b, tmp_path, rng):
    x = rng.exponential(1.0, size=(403, 5)) + rng.standard_normal((403, 5))
    port = _free_port()
    mp.spawn(_worker, args=(world, port, x, m_max, b, str(tmp_path / "out"), mode), nprocs=world, join=True)
    c1, want = orc.cumulants_upto(x, m_max, b)
    for r in range(world):
        got = np.load(tmp_path / f"out_{r}.npz")
        np.testing.assert_allclose(got["mean"], c1, rtol=1e-13)
        for k in range(2, m_max + 1):
            np.testing.assert_allclose(got[f"c{k}"], want[k], rtol=1e-9, atol=1e-12)
