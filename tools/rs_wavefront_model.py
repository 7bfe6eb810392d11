"""Shared-memory wavefront model of the streamed order-6 recursion (K3 v7/v8/v9),
calibrated on ncu's per-instruction "L1 Wavefronts Shared" of the v7d and v8
kernels (profiles/r02_rs_v7d_v8_v9_ncu.txt, profiles/r02_rs_wavefront_rule.txt).
An LDS.64 warp instruction takes

    bank rule over all 32 lanes                     if every lane quad reads <= 2 distinct addresses,
    bank rule(lanes 0-15) + bank rule(lanes 16-31)  otherwise

wavefronts (bank rule: the most distinct 4-byte words mapped to one of the 32
banks).  The quad condition is what the measurement adds: a factor whose
address depends on BOTH lane bits 0 and 1 costs 2 wavefronts even when the
whole warp reads only 4 distinct doubles, and the two half-warps are then
served separately, each with its own bank conflicts.  The rule reproduces,
exactly: v7d's 364 factor loads (157 x 1, 36 x 4/3, 171 x 2 = 547 wavefronts
per warp and unit) and its ring loads (2 each); v8's factor loads (317 x 1,
47 x 2 = 411) and its ring loads (4 each: the sub-slab and the mode-2 low bit
share a quad and the sub-slab stride is 0 mod 16 banks).

A configuration is a register tile (digits per mode a thread holds, their
digit stride) and a list of thread-level coordinates (mode, radix, digit
weight), fastest lane coordinate first.

    python tools/rs_wavefront_model.py            # the shipped kernels
    python tools/rs_wavefront_model.py --search   # lane orders of the 27-element tile
"""

import itertools
import sys

B = 6
M = 6


def terms():
    return [s for s in range(1, 1 << M, 2) if 2 <= bin(s).count("1") <= M - 2]


def stride_in(mask, q):
    later = sum(1 for p in range(q + 1, 16) if mask >> p & 1)
    return B ** later


def seg_offsets():
    """(ou, ov): offsets (doubles) of each term's first-factor slice in U and
    second factor in V (Geo::ou / Geo::ov of recursion_stream.cu)."""
    ov, ou, o1, o2 = [], [], 0, 0
    for s in terms():
        ou.append(o1)
        ov.append(o2)
        o1 += B ** (bin(s).count("1") - 1)
        o2 += B ** (M - bin(s).count("1"))
    return ou, ov


SEGV = sum(B ** (M - bin(s).count("1")) for s in terms())


def bank_rule(addrs, width=8):
    banks = {}
    for a in set(addrs):
        for w in range(width // 4):
            word = a // 4 + w
            banks.setdefault(word % 32, set()).add(word)
    return max(len(v) for v in banks.values())


def lds_wavefronts(addrs, width=8):
    quad = max(len(set(addrs[i:i + 4])) for i in range(0, len(addrs), 4))
    if quad <= 2:
        return bank_rule(addrs, width)
    return bank_rule(addrs[:16], width) + (bank_rule(addrs[16:], width) if len(addrs) > 16 else 0)


def ring_wavefronts(reg, coords):
    """Wavefronts per ring load (a thread's M_6 elements of one unit, row-major over modes 1..5)."""
    thr = threads_of(coords)
    nwarps = (len(thr) + 31) // 32
    regq = sorted(reg)
    tot, n = 0, 0
    for cmb in itertools.product(*[range(reg[q][0]) for q in regq]):
        for w in range(nwarps):
            addrs = []
            for t in thr[32 * w: 32 * w + 32]:
                off = 0
                for q in range(1, 6):
                    off += (t[q] + (reg[q][1] * cmb[regq.index(q)] if q in reg else 0)) * B ** (5 - q)
                addrs.append(8 * off)
            tot += lds_wavefronts(addrs)
            n += 1
    return tot / n


def threads_of(coords):
    """coords: [(mode, radix, weight)], fastest first -> per-thread digit base per mode."""
    n = 1
    for _, r, _ in coords:
        n *= r
    out = []
    for t in range(n):
        d = {q: 0 for q in range(1, 6)}
        x = t
        for q, r, w in coords:
            d[q] += (x % r) * w
            x //= r
        out.append(d)
    return out


def evaluate(reg, coords, detail=False):
    """reg: {mode: (count, stride)} register digits (digit = base + stride * d);
    returns (thread loads per FMA, factor-load wavefronts per element, threads, tile)."""
    ou, ov = seg_offsets()
    thr = threads_of(coords)
    nthr = len(thr)
    nelem = 1
    for q in reg:
        nelem *= reg[q][0]
    nwarps = (nthr + 31) // 32
    tot_w, tot_loads = 0, 0
    rows = []
    for ti, s in enumerate(terms()):
        r = 63 & ~s
        for kind, mask, base in (("U", s, SEGV + ou[ti]), ("V", r, ov[ti])):
            qs = [q for q in range(1, 6) if mask >> q & 1]
            regq = [q for q in qs if q in reg]
            combos = list(itertools.product(*[range(reg[q][0]) for q in regq]))
            tot_loads += len(combos)
            wsum = 0
            for cmb in combos:
                for w in range(nwarps):
                    addrs = []
                    for t in thr[32 * w: 32 * w + 32]:
                        off = base
                        for q in qs:
                            dg = t[q] + (reg[q][1] * cmb[regq.index(q)] if q in reg else 0)
                            off += dg * stride_in(mask, q)
                        addrs.append(8 * off)
                    wsum += lds_wavefronts(addrs)
            tot_w += wsum
            rows.append((ti, kind, qs, len(combos), wsum / (len(combos) * nwarps)))
    res = (tot_loads / (25.0 * nelem), tot_w / (nthr * nelem), nthr, nelem)
    return (res, rows) if detail else res


def store_sectors(reg, coords):
    """32-byte sectors touched per warp store instruction (C_6 element stores,
    row-major over modes 1..5 of one slab), averaged: 8 = fully coalesced."""
    thr = threads_of(coords)
    nwarps = (len(thr) + 31) // 32
    tot = 0
    for w in range(nwarps):
        sec = set()
        for t in thr[32 * w: 32 * w + 32]:
            off = sum(t[q] * B ** (5 - q) for q in range(1, 6))
            sec.add(off // 4)
        tot += len(sec)
    return tot / nwarps


V7D = dict(reg={3: (3, 2), 4: (3, 2), 5: (3, 2)},
           coords=[(5, 2, 1), (4, 2, 1), (3, 2, 1), (2, 6, 1), (1, 2, 1)])
# v8 / v9 (chosen by --search): lane bits 0, 1 = low bit of the mode-2 digit, sub-slab;
# bits 2..4 = group bits of modes 5, 4, 3; warp = high part of the mode-2 digit
V8 = dict(reg={3: (3, 2), 4: (3, 2), 5: (3, 2)},
          coords=[(2, 2, 1), (1, 2, 1), (5, 2, 1), (4, 2, 1), (3, 2, 1), (2, 3, 2)])

if __name__ == "__main__":
    for name, cfg in (("v7d", V7D), ("v8", V8)):
        r = evaluate(cfg["reg"], cfg["coords"])
        print(f"{name}: loads/FMA {r[0]:.3f}  factor wavefronts/element {r[1]:.4f}  threads {r[2]}  tile {r[3]}"
              f"  ring-load wavefronts {ring_wavefronts(cfg['reg'], cfg['coords']):.1f}"
              f"  store sectors/instr {store_sectors(cfg['reg'], cfg['coords']):.1f}")
    if "--search" in sys.argv:
        reg = V7D["reg"]
        # thread coordinates: group bits of modes 3, 4, 5, mode 2 as 2 x 3 or 3 x 2 or 6, sub-slab bit
        variants = {
            "tm6": [(5, 2, 1), (4, 2, 1), (3, 2, 1), (2, 6, 1), (1, 2, 1)],
            "tm2x3": [(5, 2, 1), (4, 2, 1), (3, 2, 1), (2, 2, 1), (2, 3, 2), (1, 2, 1)],
            "tm3x2": [(5, 2, 1), (4, 2, 1), (3, 2, 1), (2, 3, 1), (2, 2, 3), (1, 2, 1)],
        }
        best = []
        for vn, cs in variants.items():
            for perm in itertools.permutations(cs):
                r = evaluate(reg, list(perm))
                # factor loads + the 27 ring loads, per element
                best.append((r[1] + ring_wavefronts(reg, list(perm)) / 32.0, store_sectors(reg, list(perm)), vn, perm))
        best.sort(key=lambda x: (x[0], x[1]))
        for b in best[:25]:
            print(f"{b[0]:.4f} sectors {b[1]:.1f} {b[2]} {b[3]}")
