"""Counter-based random matrix Omega for Algorithm 1 line 1 ("Y = K_blk(Omega)
with a random Omega"; L384 "generated in a single kernel").  TEST INFRA.

Reading (R8): the paper only asks for "a random matrix".  Omega is i.i.d. with the
centred, scaled binomial distribution  Omega = (B - 32) / 4,  B ~ Binomial(64, 1/2): mean 0,
variance 1, sub-Gaussian, values in {-8, -7.75, ..., 8} -- exactly representable, so the CPU
oracle and the GPU produce bit-identical Omega, and the GPU sketch can multiply it exactly on the
int8 tensor cores.  Entry (i, j) (i = tree-order row, j = global sample column) comes from one
Philox4x32-10 block (Salmon et al., SC'11, "Parallel random numbers: as easy as 1, 2, 3"):
  counter = (i, j // 2, stream, 0),  key = (seed mod 2^32, seed >> 32),
  Omega(i, 2q)   = (popcount(w0) + popcount(w1) - 32) / 4,
  Omega(i, 2q+1) = (popcount(w2) + popcount(w3) - 32) / 4.
The CUDA path implements the same generator independently (csrc/sketch.cu).
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


def binomial_block(seed: int, stream: int, row0: int, nrows: int, col0: int, ncols: int) -> np.ndarray:
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
    pc = np.bitwise_count(w).astype(np.int64)
    g0 = (pc[0] + pc[1] - 32).astype(np.float64) / 4.0
    g1 = (pc[2] + pc[3] - 32).astype(np.float64) / 4.0
    g = np.empty((nrows, (q1 - q0) * 2))
    g[:, 0::2] = g0.reshape(nrows, q1 - q0)
    g[:, 1::2] = g1.reshape(nrows, q1 - q0)
    off = col0 - 2 * q0
    return np.ascontiguousarray(g[:, off:off + ncols])


# the Omega stream used by Algorithm 1 (R8)
omega_block = binomial_block
