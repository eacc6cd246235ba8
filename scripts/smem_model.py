"""Shared-memory wavefront model of the tile decoder's access patterns.

For a sample of real tiles (c1, c2, c4 streams), counts the wavefronts each
warp-wide shared-memory instruction needs (max lanes per bank, in 4-byte
words; vector accesses split into 128-byte wavefront groups) for the
candidate layouts, so swizzles can be chosen before touching the kernel.
Usage: python scripts/smem_model.py
"""
import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1503_07387_b200 import workload as W  # noqa: E402


def wavefronts(word_addrs, width_words=1):
    """Wavefronts for one warp instruction: lanes' starting word addresses
    (None = inactive), each accessing `width_words` consecutive words."""
    acc = [a for a in word_addrs if a is not None]
    if not acc:
        return 0
    if width_words == 1:
        banks = {}
        seen = set()
        for a in acc:
            if a in seen:
                continue  # same word: broadcast
            seen.add(a)
            banks[a % 32] = banks.get(a % 32, 0) + 1
        return max(banks.values())
    # vector: process in groups of 32/width lanes per wavefront minimum
    per = 32 // width_words
    total = 0
    for g in range(0, len(acc), per):
        grp = acc[g:g + per]
        banks = {}
        for a in grp:
            for k in range(width_words):
                b = (a + k) % 32
                banks[b] = banks.get(b, 0) + 1
        total += max(banks.values())
    return total


def swz(kind, w):
    if kind == "none":
        return w
    if kind == "x2_5":   # word bits 2-3 ^= bits 5-6
        return w ^ ((w >> 3) & 0xC)
    if kind == "x3_5":   # bits 2-4 ^= bits 5-7
        return w ^ ((w >> 3) & 0x1C)
    if kind == "x4_5":   # bits 2-5 ^= bits 6-9 (keeps 16-B chunks)
        return w ^ ((w >> 4) & 0x3C)
    raise ValueError(kind)


def tile_ends(enc, t, tile=4096):
    seg = enc[t * tile:(t + 1) * tile]
    return np.flatnonzero(seg < 0x80)


def model(name, enc, tiles, ints_per_lane=8, swizzles=("none", "x2_5", "x3_5", "x4_5")):
    res = {s: {"V_st": 0, "V_gather": 0} for s in swizzles}
    ep = {"EP_scatter": 0, "EP_scatter_pad": 0, "EP_load": 0, "EP_load_pad": 0}
    n_tiles = 0
    for t in tiles:
        ends = tile_ends(enc, t)
        n = ends.size
        lp_end = ends + 16  # local coords
        starts = np.concatenate([[15], lp_end[:-1]]) + 1
        n_tiles += 1
        for s in swizzles:
            # V stores: lane l (tid) writes words 16+16l+4j .. +3, j = 0..3 (STS.128)
            for w in range(8):
                for j in range(4):
                    addrs = [swz(s, 16 + 16 * (32 * w + l) + 4 * j) for l in range(32)]
                    res[s]["V_st"] += wavefronts(addrs, 4)
            # V gather: phase-2 lane u handles ints [k*u, k*u+k), pass structure ignored
            k = ints_per_lane
            lanes = (n + k - 1) // k
            for w in range((lanes + 31) // 32):
                for j in range(k):
                    addrs = []
                    for l in range(32):
                        u = 32 * w + l
                        i = k * u + j
                        addrs.append(swz(s, int(starts[i])) if i < n else None)
                    res[s]["V_gather"] += wavefronts(addrs, 1)
        # EP scatter: chunk lanes, position j instruction, rank address
        T = np.zeros(4096, bool)
        T[ends] = True
        cnt = T.reshape(256, 16).sum(1)
        excl = np.concatenate([[0], np.cumsum(cnt)[:-1]])
        for w in range(8):
            for j in range(16):
                a1, a2 = [], []
                for l in range(32):
                    c = 32 * w + l
                    if T[16 * c + j]:
                        r = excl[c] + T[16 * c:16 * c + j].sum()
                        a1.append(4 + int(r))
                        a2.append(4 + int(r) + 4 * (int(r) >> 4))
                    else:
                        a1.append(None)
                        a2.append(None)
                ep["EP_scatter"] += wavefronts(a1)
                ep["EP_scatter_pad"] += wavefronts(a2)
        # EP loads: lane u reads k entries starting 4 + k*u (vector 4 words)
        k = ints_per_lane
        lanes = (n + k - 1) // k
        for w in range((lanes + 31) // 32):
            for q in range(k // 4):
                a1 = [4 + k * (32 * w + l) + 4 * q for l in range(32)]
                a2 = [4 + (k * (32 * w + l) + 4 * q) + 4 * ((k * (32 * w + l) + 4 * q) >> 4) for l in range(32)]
                ep["EP_load"] += wavefronts(a1, 4)
                ep["EP_load_pad"] += wavefronts(a2, 4)
    print(f"== {name}: {n_tiles} tiles, ints/lane {ints_per_lane}, per tile wavefronts")
    for s in swizzles:
        print(f"   V[{s:5s}] store {res[s]['V_st'] / n_tiles:7.1f}   gather {res[s]['V_gather'] / n_tiles:7.1f}")
    for k_, v in ep.items():
        print(f"   {k_:15s} {v / n_tiles:7.1f}")


def main():
    rng_tiles = range(100, 116)
    for name, mk in (("c1", lambda: W.config1(1 << 20)), ("c2", lambda: W.config2(1 << 20)),
                     ("c4", lambda: W.config4(1 << 20))):
        w = mk()
        for k in (8, 16):
            model(name, w.encoded, rng_tiles, ints_per_lane=k)


if __name__ == "__main__":
    main()
