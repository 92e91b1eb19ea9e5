"""Philox4x32-10 counter-based RNG, NumPy, for the dropout mask (reading C14).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper fixes no dropout RNG (App. B row "Dropout", P:L1295-1296 gives
shapes only).  DESIGN.md reading R14: the mask bit of element i of model b at
step t in dropout layer `layer` is drawn from Philox4x32-10 (Salmon et al.,
SC'11) with counter (i // 4, b, t, layer), key (seed mod 2^32, seed >> 32),
output word i % 4; the element is KEPT iff word >= floor(p * 2^32).  The CUDA
path implements the same generator independently (csrc), so masks are
bit-identical and parity is exact.

Pinned by the Random123 known-answer vectors in tests/golden/philox_kat.txt.
"""
import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr, key):
    """ctr: 4 uint arrays (broadcastable), key: 2 ints -> 4 uint64 arrays of u32 words."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) & MASK for c in ctr)
    k0, k1 = int(key[0]) & 0xFFFFFFFF, int(key[1]) & 0xFFFFFFFF
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & 0xFFFFFFFF
            k1 = (k1 + W1) & 0xFFFFFFFF
        p0 = M0 * c0            # < 2^64: exact in uint64
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0), lo1,
                          hi0 ^ c3 ^ np.uint64(k1), lo0)
    return c0, c1, c2, c3


def keep_threshold(p):
    """floor(p * 2^32) computed from float32(p), saturated to 2^32 - 1."""
    t = np.floor(np.float64(np.float32(p)) * 4294967296.0)
    return int(min(t, 4294967295.0))


def dropout_keep_mask(seed, b, step, layer, n_elem, p):
    """Boolean keep-mask of n_elem elements (row-major over the model's tensor)."""
    i = np.arange(n_elem, dtype=np.uint64)
    words = philox4x32_10((i // np.uint64(4), np.full_like(i, b), np.full_like(i, step),
                           np.full_like(i, layer)),
                          (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF))
    w = np.stack(words, axis=0)              # [4, n]
    sel = w[(i % np.uint64(4)).astype(np.int64), np.arange(n_elem)]
    return sel >= np.uint64(keep_threshold(p))
