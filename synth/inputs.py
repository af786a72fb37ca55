"""Seeded synthetic inputs with the shapes of the paper's workloads.

- uniform_points: i.i.d. U[0,1)^dim ("uniform 3D distribution of points in a cube").
- grid_points: cell-centred regular grid (BASELINE.json configs[3]: volume IE on a regular grid;
  SURVEY.md Z22: 128x128x64 cells of spacing 1/128 for N=2^20).
- probe_vectors: Gaussian N x q block used only for a-posteriori error probes.
"""
import numpy as np

__all__ = ["uniform_points", "grid_points", "probe_vectors", "lowrank_factor", "workload", "WORKLOADS"]


def uniform_points(n: int, dim: int = 3, seed: int = 0) -> np.ndarray:
    """n x dim float64, row-major, i.i.d. uniform in [0,1)^dim (numpy PCG64, given seed)."""
    if n < 1 or dim not in (1, 2, 3):
        raise ValueError("uniform_points: need n >= 1 and dim in {1,2,3}")
    return np.random.default_rng(seed).random((n, dim))


def grid_points(shape, spacing: float) -> np.ndarray:
    """Cell-centred grid: point (i,j,k) = ((i+0.5)h, (j+0.5)h, (k+0.5)h); x fastest-varying last.

    Returned n x dim in C order over (i, j, k) so that the last axis varies fastest.
    """
    axes = [(np.arange(s, dtype=np.float64) + 0.5) * spacing for s in shape]
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([m.reshape(-1) for m in mesh], axis=1).copy()


def probe_vectors(n: int, q: int = 16, seed: int = 2) -> np.ndarray:
    """n x q float64 standard normal probe block (probe seed 2)."""
    return np.random.default_rng(seed).standard_normal((n, q))


def lowrank_factor(n: int, r: int = 64, seed: int = 3) -> np.ndarray:
    """n x r float64 factor U of the symmetric update U U^T (BASELINE configs[4], R24):
    i.i.d. N(0, 1/r), so diag(U U^T) ~ 1 like the covariance diagonal."""
    return np.random.default_rng(seed).standard_normal((n, r)) / np.sqrt(r)


# name -> (points factory, kernel kind, kernel parameter, leaf size, tol)
# kernel kinds: "exp" = e^{-r/l} (PAPER.md Eq. cov), "helmholtz" = cos(k r)/r, 0 on the
# diagonal (PAPER.md Eq. ie).
WORKLOADS = {
    # BASELINE.json configs[0]: 2D exp covariance, N=1024 uniform, leaf 32, tol 1e-6
    "cov2d_1k": dict(points=lambda: uniform_points(1024, 2, 0), kernel="exp", param=0.2, leaf=32, tol=1e-6),
    # BASELINE.json configs[1]: 3D covariance, N=2^18 uniform, leaf 64, tol 1e-6, dense-kernel sketch
    "cov3d_256k": dict(points=lambda: uniform_points(1 << 18, 3, 0), kernel="exp", param=0.2, leaf=64, tol=1e-6),
    # BASELINE.json configs[2]: 3D exp covariance, N=2^21
    # S§8(f) NEXT #1 at N = 2^20 (the O(N) H^2-matvec sketch of a bootstrap H^2; tools/run_config.py --bootstrap)
    "cov3d_1m": dict(points=lambda: uniform_points(1 << 20, 3, 0), kernel="exp", param=0.2, leaf=64, tol=1e-6),
    "cov3d_2m": dict(points=lambda: uniform_points(1 << 21, 3, 0), kernel="exp", param=0.2, leaf=64, tol=1e-6),
    # BASELINE.json configs[3]: volume IE cos(3r)/r on a 128x128x64 grid (N=2^20), tol 1e-4
    "ie3d_1m": dict(points=lambda: grid_points((128, 128, 64), 1.0 / 128), kernel="helmholtz", param=3.0,
                    leaf=64, tol=1e-4),
    # BASELINE configs[4]: recompress H2(A) + U U^T, A = exp covariance H^2 (tol 1e-6), rank-64 update
    "h2update_1m": dict(points=lambda: uniform_points(1 << 20, 3, 0), kernel="exp", param=0.2, leaf=64, tol=1e-6,
                        update_rank=64, d_max=1024, p_os=32),
    # configs[4] shape at N = 2^18 (the U V^T update of h2_build_nonsym stores every ordered block)
    "h2update_256k": dict(points=lambda: uniform_points(1 << 18, 3, 0), kernel="exp", param=0.2, leaf=64, tol=1e-6,
                          update_rank=64, d_max=1024, p_os=32),
    # small parity cases (ragged sizes, several tiles)
    "cov3d_5k": dict(points=lambda: uniform_points(5000, 3, 0), kernel="exp", param=0.2, leaf=64, tol=1e-6),
    "ie3d_4k": dict(points=lambda: grid_points((16, 16, 16), 1.0 / 16), kernel="helmholtz", param=3.0,
                    leaf=64, tol=1e-4),
    # an explicit dense operator (frontal-matrix stand-in) -- the exp kernel
    # matrix materialised on the GPU in tree order; sketch = DGEMM, entries = lookups
    "dense_op_32k": dict(points=lambda: uniform_points(1 << 15, 3, 0), kernel="exp", param=0.2, leaf=64, tol=1e-6,
                         dense=True),
    "dense_op_64k": dict(points=lambda: uniform_points(1 << 16, 3, 0), kernel="exp", param=0.2, leaf=64, tol=1e-6,
                         dense=True),
}


def workload(name: str):
    w = dict(WORKLOADS[name])
    w["points"] = w["points"]()
    return w
