"""Randomized parity sweep: random (n, m, b, t, distribution) through the
GPU path (moment, cumulants_upto, moment_parallel_blocks, outer_prod_cum)
against the CPU oracle.  Prints one line per failure and a summary.
Moments: rtol 1e-12; cumulants: |got - want| <= 1e-9 |want| + 1e-11 x the
magnitude of the terms the recursion subtracts (cancellation-aware).

    python tools/fuzz_parity.py --cases 300 --seed 1
"""

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1701_05420_b200 as bcg  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def draw(rng, t, n):
    kind = rng.integers(0, 4)
    if kind == 0:
        return rng.standard_normal((t, n))
    if kind == 1:
        return rng.exponential(1.0, (t, n)) * rng.uniform(0.1, 10.0, n)
    if kind == 2:
        return rng.standard_t(5, (t, n)) + rng.uniform(-100, 100, n)
    return np.round(rng.standard_normal((t, n)) * 4) / 4  # ties / exact small values


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=200)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--wide", action="store_true", help="wide matrices: n up to 400 (m=2), 120 (m=3), 40 (m=4)")
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    fails = 0
    t0 = time.time()
    for case in range(a.cases):
        m = int(rng.integers(2, 5 if a.wide else 9))
        b = int(rng.integers(1, 17 if a.wide else 9))
        nmax = {2: 400, 3: 120, 4: 40} if a.wide else {2: 70, 3: 40, 4: 24, 5: 14, 6: 10, 7: 7, 8: 5}
        n = int(rng.integers(1, nmax[m]))
        # a quarter of the cases span several 16384-sample split-K slices
        t = int(rng.integers(2, 3000)) if rng.random() < 0.75 or m > 4 else int(rng.integers(16000, 70000))
        x = draw(rng, t, n)
        what = f"case {case}: n={n} m={m} b={b} t={t}"
        try:
            got = bcg.moment(x, m, b).packed_host()
            np.testing.assert_allclose(got, orc.moment(x, m, b), rtol=1e-12, atol=1e-13 * max(1.0, np.abs(x).max() ** m))
            p = int(rng.integers(2, 5))
            np.testing.assert_array_equal(bcg.moment_parallel_blocks(x, m, b, p=p).packed_host(), got)
            cs = bcg.cumulants_upto(x, m, b=b)
            c1, want = orc.cumulants_upto(x, m, b)
            np.testing.assert_allclose(cs[1], c1, rtol=1e-12, atol=1e-12)
            # an element's rounding error scales with the magnitudes its
            # computation cancels: the sample sum's absolute moment
            # (1/t) sum_l prod |x_c| plus, from order 4, the reference's
            # partition sums of |lower cumulants| (bc/cumulants.py:53-136) --
            # not with |C_k| itself
            xc = x - x.mean(axis=0)
            for k in range(2, m + 1):
                w = want[k]
                term = orc.moment(np.abs(xc), k, b)
                if k >= 4:
                    absl = {j: np.abs(want[j]) for j in range(2, k - 1)}
                    for sigma in range(2, k // 2 + 1):
                        term = term + orc.outer_prod_cum(k, sigma, absl, n, b)
                err = np.abs(cs[k].packed_host() - w)
                bad = err > 1e-9 * np.abs(w) + 1e-11 * term + 1e-300
                if bad.any():
                    i = int(np.argmax(bad))
                    raise AssertionError(f"C{k}: {int(bad.sum())} elements, e.g. [{i}] got-want {err[i]:.3e} "
                                         f"|want| {abs(w[i]):.3e} term scale {term[i]:.3e}")
        except Exception as exc:  # report and continue
            fails += 1
            msg = " | ".join(line.strip() for line in str(exc).splitlines() if line.strip())
            print(f"FAIL {what}: {type(exc).__name__}: {msg[:600]}", flush=True)
    print(f"{a.cases} cases, {fails} failures, {time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    main()
