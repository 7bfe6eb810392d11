"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container (where /root/reference exists):

    ./oracle/build_ref.sh            # builds the unmodified reference into oracle/_ref
    python tests/golden/make_golden.py

It imports the reference package ``blockcumulants`` (compiled engine, its
default ``engine="auto"``) from oracle/_ref and records its outputs on seeded
inputs.  The fixtures are committed; /root/reference never travels to the GPU
box, so the tests read only these files.

Contents (all float64 values are the reference's own results):

* ``layout.npz``   -- ``_block_layout`` tables (bc/_engines.py:46-54) for small
                      (n, m, b) incl. partial edges, and SHA-256 digests of the
                      tables for every BASELINE config and order 2..m.
* ``partitions.json`` -- ``enumerate_partitions_min2`` (bc/partitions.py:63-98)
                      for m = 2..8 in the reference's order.
* ``moments.npz``  -- ``moment(x, m, b)`` packed, on the reference's own test
                      grid (pkg/tests/test_moments.py:116-126), inputs stored.
* ``cumulants.npz`` -- ``cumulants_upto(x, m_max, b)`` packed C1..C_m for a grid
                      following pkg/tests/test_acceptance.py:44-66 (+ partial
                      edges), inputs stored.
* ``configs.npz``  -- the BASELINE recipes at reduced t (workloads.py): X and a
                      seeded sample of 4096 packed positions per order of the
                      reference's cumulants, plus per-order sum/sum-of-squares;
                      cfg1 at its full size (X regenerated from the recipe).
* ``highorder.npz`` -- heavy-tailed data to order 6 (the Student-t(5)
                      copula of cfg2 / cfg5, whose 6th moment does not exist:
                      the sample cumulants cancel hardest there): the cfg5
                      recipe's first 36 columns at b=6 and the cfg2 recipe's
                      first 32 columns at b=8, t=3000 rows, m=6.  Stored: a
                      checksum of X, 4096 sampled packed positions per order,
                      and per-BLOCK sums / sums of squares of every C_k (a
                      checksum of checksums over all 21.6 M / 22.0 M elements
                      of C_6).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
sys.path.insert(0, ROOT)

import blockcumulants as bc  # noqa: E402  (the reference)
from blockcumulants import _engines  # noqa: E402
from blockcumulants.partitions import enumerate_partitions_min2  # noqa: E402

import workloads  # noqa: E402

assert bc.HAVE_COMPILED, "reference _core not built; run oracle/build_ref.sh"


def packed(tensor) -> np.ndarray:
    """Concatenate blocks in lexicographic key order (the reference's flat
    buffer order, bc/_engines.py:57-61)."""
    keys = sorted(tensor.blocks)
    return np.concatenate([tensor.blocks[k].ravel(order="C") for k in keys])


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def layout_fixture():
    out = {}
    small = [(5, 3, 2), (7, 4, 3), (3, 3, 5), (2, 6, 1), (6, 6, 2), (24, 4, 4),
             (5, 2, 2), (9, 5, 4), (10, 1, 3)]
    for n, m, b in small:
        keys, col0, edges, offs = _engines._block_layout(n, m, b)
        tag = f"{n}_{m}_{b}"
        out[f"keys_{tag}"] = np.array(keys, dtype=np.int64).reshape(len(keys), m)
        out[f"col0_{tag}"] = col0
        out[f"edges_{tag}"] = edges
        out[f"offs_{tag}"] = offs
    digests = {}
    for name, cfg in workloads.CONFIGS.items():
        for m in range(2, cfg.m + 1):
            keys, col0, edges, offs = _engines._block_layout(cfg.n, m, cfg.b)
            karr = np.array(keys, dtype=np.int64).reshape(len(keys), m)
            digests[f"{cfg.n}_{m}_{cfg.b}"] = sha(karr, col0, edges, offs)
    out["digests"] = np.array(json.dumps(digests))
    np.savez_compressed(os.path.join(HERE, "layout.npz"), **out)


def partitions_fixture():
    table = {}
    for m in range(2, 9):
        for sigma in range(2, m // 2 + 1):
            table[f"{m},{sigma}"] = [list(map(list, p)) for p in enumerate_partitions_min2(m, sigma)]
    with open(os.path.join(HERE, "partitions.json"), "w") as f:
        json.dump(table, f, separators=(",", ":"))


MOMENT_GRID = [(4, 3, 2, 100), (5, 4, 2, 60), (5, 4, 3, 60), (3, 5, 2, 40),
               (6, 2, 4, 200), (2, 6, 1, 30), (3, 3, 5, 50), (6, 6, 2, 300),
               (7, 4, 3, 257), (12, 5, 4, 1000), (9, 6, 3, 400)]


def moments_fixture():
    out = {}
    for i, (n, m, b, t) in enumerate(MOMENT_GRID):
        rng = np.random.default_rng(1000 + i)
        x = rng.standard_normal((t, n))
        out[f"x_{i}"] = x
        out[f"m_{i}"] = packed(bc.moment(x, m, b))
        out[f"shape_{i}"] = np.array([n, m, b, t], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "moments.npz"), **out)


CUM_GRID = []
for n in (2, 3, 4, 5):
    for t in (100, 1000):
        for dist in ("gaussian", "uniform", "exponential"):
            CUM_GRID.append((n, t, dist, 1 + len(CUM_GRID) % 3, 6, 2))
CUM_GRID += [(5, 400, "exponential", 7, 6, 3), (7, 500, "uniform", 8, 5, 3),
             (6, 300, "gaussian", 9, 6, 4), (8, 800, "exponential", 10, 4, 3)]


def cumulants_fixture():
    from blockcumulants import dataio

    out = {}
    for i, (n, t, dist, seed, m_max, b) in enumerate(CUM_GRID):
        x = dataio.generate(dist, n, t, seed=seed)
        cs = bc.cumulants_upto(x, m_max, b=b)
        out[f"x_{i}"] = x
        out[f"c1_{i}"] = cs[1]
        for k in range(2, m_max + 1):
            out[f"c{k}_{i}"] = packed(cs[k])
        out[f"shape_{i}"] = np.array([n, t, m_max, b], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "cumulants.npz"), **out)


CONFIG_T = {"cfg2": 1000, "cfg3": 600, "cfg4": 500, "cfg5": 150}
# cfg5 at order 5/6 is 1.2e8 / 2.5e9 stored elements: beyond the CPU
# reference's reach; its fixture stops at order 4.
CONFIG_M = {"cfg5": 4}


def configs_fixture():
    out = {}
    for name, cfg in workloads.CONFIGS.items():
        t = cfg.t if name == "cfg1" else CONFIG_T[name]
        m_top = CONFIG_M.get(name, cfg.m)
        x = workloads.generate(name, t)
        cs = bc.cumulants_upto(x, m_top, b=cfg.b)
        if name != "cfg1":
            out[f"{name}_x"] = x
        else:
            out[f"{name}_xsum"] = np.array([x.sum(), (x * x).sum()])
        out[f"{name}_c1"] = cs[1]
        print("  ", name, "done", flush=True)
        rng = np.random.default_rng(99)
        for k in range(2, m_top + 1):
            flat = packed(cs[k])
            idx = np.sort(rng.choice(flat.size, size=min(4096, flat.size), replace=False))
            out[f"{name}_c{k}_idx"] = idx.astype(np.int64)
            out[f"{name}_c{k}_val"] = flat[idx]
            out[f"{name}_c{k}_stats"] = np.array([flat.sum(), (flat * flat).sum(), flat.size])
    np.savez_compressed(os.path.join(HERE, "configs.npz"), **out)


# (config recipe, columns kept, b, t, m): heavy tails to order 6 within the
# CPU reference's reach (C_6 of 21-22 M elements)
HIGHORDER = {"cfg5s": ("cfg5", 36, 6, 3000, 6), "cfg2s": ("cfg2", 32, 8, 3000, 6)}


def highorder_input(tag: str) -> np.ndarray:
    name, ncols, _, t, _ = HIGHORDER[tag]
    return np.ascontiguousarray(workloads.generate(name, t)[:, :ncols])


def highorder_fixture():
    out = {}
    for tag, (name, ncols, b, t, m) in HIGHORDER.items():
        x = highorder_input(tag)
        cs = bc.cumulants_upto(x, m, b=b)
        out[f"{tag}_xsum"] = np.array([x.sum(), (x * x).sum(), np.abs(x).max()])
        out[f"{tag}_c1"] = cs[1]
        rng = np.random.default_rng(123)
        for k in range(2, m + 1):
            flat = packed(cs[k])
            idx = np.sort(rng.choice(flat.size, size=min(4096, flat.size), replace=False))
            out[f"{tag}_c{k}_idx"] = idx.astype(np.int64)
            out[f"{tag}_c{k}_val"] = flat[idx]
            blocks = list(cs[k].blocks.values())
            out[f"{tag}_c{k}_bsum"] = np.array([blk.sum() for blk in blocks])
            out[f"{tag}_c{k}_bsq"] = np.array([(blk * blk).sum() for blk in blocks])
            out[f"{tag}_c{k}_bmax"] = np.array([np.abs(blk).max() for blk in blocks])
        print("  ", tag, "done", flush=True)
    np.savez_compressed(os.path.join(HERE, "highorder.npz"), **out)


if __name__ == "__main__":
    import time

    only = sys.argv[1:]
    for fn in (layout_fixture, partitions_fixture, moments_fixture,
               cumulants_fixture, configs_fixture, highorder_fixture):
        if only and fn.__name__ not in only:
            continue
        t0 = time.time()
        fn()
        print(fn.__name__, f"{time.time() - t0:.1f}s", flush=True)
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))
