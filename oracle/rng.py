"""Counter-based Gaussian random matrix Omega for Algorithm 1 line 1 (PAPER.md L203,
"Y = K_blk(Omega) with a random Omega"; L384 "generated in a single kernel").  TEST INFRA.

Reading (R8): Omega is i.i.d. standard normal.  Entry (i, j) of the stream
(i = tree-order row, j = global sample column) is produced from one Philox4x32-10 block
(Salmon et al., SC'11, "Parallel random numbers: as easy as 1, 2, 3") with
  counter = (i, j // 2, stream, 0),  key = (seed mod 2^32, seed >> 32)
whose 4 words give two 53-bit uniforms u1 = ((w1:w0) >> 11 + 0.5) 2^-53 and
u2 = ((w3:w2) >> 11 + 0.5) 2^-53, and the Box-Muller pair
  Omega(i, 2q)   = sqrt(-2 ln u1) cos(2 pi u2),
  Omega(i, 2q+1) = sqrt(-2 ln u1) sin(2 pi u2).
The CUDA path implements the same generator independently (csrc/rand.cu).
"""
import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = np.uint32(0x9E3779B9)
W1 = np.uint32(0xBB67AE85)
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr, key):
    """Philox4x32 with 10 rounds.  ctr: (4, n) uint32, key: (2, n) uint32 -> (4, n) uint32.

    Round (Random123 philox4x32round): hi0:lo0 = M0*c0, hi1:lo1 = M1*c2,
    c' = (hi1^c1^k0, lo1, hi0^c3^k1, lo0); the key is bumped by (W0, W1) between rounds.
    """
    c = [np.asarray(x, dtype=np.uint32).copy() for x in ctr]
    k0 = np.asarray(key[0], dtype=np.uint32).copy()
    k1 = np.asarray(key[1], dtype=np.uint32).copy()
    with np.errstate(over="ignore"):
        for r in range(10):
            if r > 0:
                k0 = (k0 + W0).astype(np.uint32)
                k1 = (k1 + W1).astype(np.uint32)
            p0 = M0 * c[0].astype(np.uint64)
            p1 = M1 * c[2].astype(np.uint64)
            hi0 = (p0 >> np.uint64(32)).astype(np.uint32)
            lo0 = (p0 & MASK32).astype(np.uint32)
            hi1 = (p1 >> np.uint64(32)).astype(np.uint32)
            lo1 = (p1 & MASK32).astype(np.uint32)
            c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
    return np.stack(c)


def _u53(lo, hi):
    v = (hi.astype(np.uint64) << np.uint64(32)) | lo.astype(np.uint64)
    return ((v >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)


def gaussian_block(seed: int, stream: int, row0: int, nrows: int, col0: int, ncols: int) -> np.ndarray:
    """Rows [row0, row0+nrows) x columns [col0, col0+ncols) of the Omega stream, float64."""
    if nrows <= 0 or ncols <= 0:
        return np.zeros((max(nrows, 0), max(ncols, 0)))
    q0, q1 = col0 // 2, (col0 + ncols + 1) // 2
    rows = np.arange(row0, row0 + nrows, dtype=np.uint64)
    qs = np.arange(q0, q1, dtype=np.uint64)
    R, Q = np.meshgrid(rows, qs, indexing="ij")
    n = R.size
    ctr = np.stack([R.reshape(-1).astype(np.uint32), Q.reshape(-1).astype(np.uint32),
                    np.full(n, stream, np.uint32), np.zeros(n, np.uint32)])
    key = np.stack([np.full(n, seed & 0xFFFFFFFF, np.uint32), np.full(n, (seed >> 32) & 0xFFFFFFFF, np.uint32)])
    w = philox4x32_10(ctr, key)
    u1 = _u53(w[0], w[1])
    u2 = _u53(w[2], w[3])
    rad = np.sqrt(-2.0 * np.log(u1))
    g0 = rad * np.cos(2.0 * np.pi * u2)
    g1 = rad * np.sin(2.0 * np.pi * u2)
    g = np.empty((nrows, (q1 - q0) * 2))
    g[:, 0::2] = g0.reshape(nrows, q1 - q0)
    g[:, 1::2] = g1.reshape(nrows, q1 - q0)
    off = col0 - 2 * q0
    return np.ascontiguousarray(g[:, off:off + ncols])
