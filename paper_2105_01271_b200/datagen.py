"""BASELINE synthetic snapshot fields.

A[i, j] = sum_modes c_mode * prod_dims sin(pi p_d x_d) * exp(-|p|^2 pi^2 nu t_i)

on the interior grid x = (1..g)/(g+1) of each dimension, t_i = linspace(0, 1, m)
(src/datagen.py:93 convention), columns flattened in C order over (x, y[, z])
with p<->x, q<->y, r<->z.  Coefficients are drawn p-major from
Philox(seed) (the reference's RNG, src/sketch.py:33-35); cfg3's noise
(variance 1e-6, i.e. std 1e-3) is drawn afterwards from the same generator.
cfg5 is generated in FP64 and rounded once to FP32.

The reference's own ``gen_heat2d`` (src/datagen.py:74-100) is a different
(periodic) field, so this module is new.  There is no public dataset: the
paper's NACA / channel / JHU data are replaced by these seeded fields.

The host generator below is BLAS-free (elementwise numpy in a fixed order), so
its bytes do not depend on the BLAS build or thread count; parity runs feed the
SAME bytes to the oracle and to the device path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class FieldConfig:
    name: str
    m: int
    grid: tuple            # points per dimension
    modes: int             # P: p, q (, r) in 1..P
    coef_power: float      # c = N(0,1) / |p|^(2*coef_power)
    nu: float
    seed: int
    stride: int            # coarse-grid stride per dimension
    k: int
    q: int                 # power iterations (0 = single_pass_svd)
    noise_std: float = 0.0
    dtype: str = "f64"

    @property
    def n(self) -> int:
        return int(np.prod(self.grid))

    @property
    def dims(self) -> int:
        return len(self.grid)

    @property
    def n_coarse(self) -> int:
        return int(np.prod([len(range(0, g, self.stride)) for g in self.grid]))

    @property
    def a_bytes(self) -> int:
        return self.m * self.n * (8 if self.dtype == "f64" else 4)

    def scaled(self, m=None, grid=None, name=None):
        return FieldConfig(name or self.name + "-scaled", m or self.m, grid or self.grid,
                           self.modes, self.coef_power, self.nu, self.seed, self.stride,
                           self.k, self.q, self.noise_std, self.dtype)


# BASELINE.json "configs" (cfg1..cfg5)
CONFIGS = {
    "cfg1": FieldConfig("cfg1", 1000, (64, 64), 5, 1.0, 0.01, 0, 4, 20, 0),
    "cfg2": FieldConfig("cfg2", 2000, (256, 256), 20, 1.0, 0.005, 1, 4, 50, 1),
    "cfg3": FieldConfig("cfg3", 5000, (512, 512), 40, 0.5, 0.001, 2, 8, 100, 1,
                        noise_std=1e-3),
    "cfg4": FieldConfig("cfg4", 10000, (1024, 1024), 60, 0.75, 0.002, 3, 8, 200, 1),
    "cfg5": FieldConfig("cfg5", 2000, (256, 256, 256), 12, 1.0, 0.003, 4, 4, 100, 1,
                        dtype="f32"),
}


def coarse_grid_indices(grid, stride) -> np.ndarray:
    """Flattened (C-order) indices of the points whose every coordinate is
    a multiple of ``stride`` -- the BASELINE coarse grid, ascending."""
    axes = [np.arange(0, g, stride, dtype=np.int64) for g in grid]
    mesh = np.meshgrid(*axes, indexing="ij")
    flat = np.zeros(mesh[0].shape, dtype=np.int64)
    for ax, g in zip(mesh, grid):
        flat = flat * g + ax
    return flat.ravel()


def mode_tables(cfg: FieldConfig):
    """(S, lam, coef): S[i_x, p-1] = sin(pi p x_i); lam and coef flattened p-major."""
    rng = np.random.Generator(np.random.Philox(cfg.seed))
    P = cfg.modes
    p = np.arange(1, P + 1, dtype=np.float64)
    grids = [np.arange(1, g + 1, dtype=np.float64) / (g + 1.0) for g in cfg.grid]
    S = [np.sin(np.pi * np.outer(x, p)) for x in grids]
    mesh = np.meshgrid(*([p] * cfg.dims), indexing="ij")
    lam = sum(mm ** 2 for mm in mesh).ravel()
    coef = rng.standard_normal(lam.size) / lam ** cfg.coef_power
    return S, lam, coef, rng


def generate_host(cfg: FieldConfig) -> np.ndarray:
    """Deterministic, BLAS-free host generator (row-major m x n)."""
    S, lam, coef, rng = mode_tables(cfg)
    t = np.linspace(0.0, 1.0, cfg.m)
    P = cfg.modes
    out = np.zeros((cfg.m,) + tuple(cfg.grid))
    if cfg.dims == 2:
        gx, gy = cfg.grid
        # out[i, x, y] += sum_p S_x[x,p] * (sum_q E[i,(p,q)] * S_y[y,q])
        for a in range(P):
            inner = np.zeros((cfg.m, gy))
            for b in range(P):
                mu = a * P + b
                e = np.exp(-lam[mu] * np.pi ** 2 * cfg.nu * t) * coef[mu]
                inner += e[:, None] * S[1][None, :, b]
            out += S[0][None, :, a, None] * inner[:, None, :]
    elif cfg.dims == 3:
        gx, gy, gz = cfg.grid
        for a in range(P):
            mid = np.zeros((cfg.m, gy, gz))
            for b in range(P):
                inner = np.zeros((cfg.m, gz))
                for c in range(P):
                    mu = (a * P + b) * P + c
                    e = np.exp(-lam[mu] * np.pi ** 2 * cfg.nu * t) * coef[mu]
                    inner += e[:, None] * S[2][None, :, c]
                mid += S[1][None, :, b, None] * inner[:, None, :]
            out += S[0][None, :, a, None, None] * mid[:, None, :, :]
    else:
        raise ValueError("only 2-D and 3-D fields")
    out = out.reshape(cfg.m, cfg.n)
    if cfg.noise_std:
        out += rng.standard_normal(out.shape) * cfg.noise_std
    if cfg.dtype == "f32":
        out = out.astype(np.float32)
    return out


def generate_device(cfg: FieldConfig, device=None, chunk_rows: int = 0, x_range=None):
    """The same field built on the GPU with FP64 GEMMs (input setup for the
    configurations too large for the host generator: cfg4 is 84 GB, cfg5
    134 GB).  Separable evaluation A[i, x, y(, z)] = sum_p Sx[x,p] T_p where
    T contracts the remaining dimensions; rows are produced in chunks so the
    FP64 intermediates stay small.  cfg3's noise is drawn on the host in row
    chunks from the same Philox stream as generate_host (same values).
    Returns a CUDA tensor (float64, or float32 for dtype "f32").

    ``x_range = (x0, x1)`` builds only the x-slab x0 <= ix < x1 of the grid
    (columns [x0*g_rest, x1*g_rest) of the full matrix): one rank's shard of
    the column-sharded layout (noise-free fields only)."""
    import torch
    dev = device or torch.device("cuda", torch.cuda.current_device())
    S, lam, coef, rng = mode_tables(cfg)
    t = np.linspace(0.0, 1.0, cfg.m)
    P = cfg.modes
    out_dtype = torch.float64 if cfg.dtype == "f64" else torch.float32
    ncols = cfg.n
    if x_range is not None:
        if cfg.noise_std:
            raise ValueError("x-slab generation is for noise-free fields")
        S = [S[0][x_range[0]:x_range[1]]] + list(S[1:])
        ncols = (x_range[1] - x_range[0]) * int(np.prod(cfg.grid[1:]))
    A = torch.empty((cfg.m, ncols), dtype=out_dtype, device=dev)
    Sd = [torch.from_numpy(np.ascontiguousarray(s)).to(dev) for s in S]
    lam_d = torch.from_numpy(lam).to(dev)
    coef_d = torch.from_numpy(coef).to(dev)
    if chunk_rows <= 0:
        per_row = cfg.n * 8 * (2 if cfg.dims == 3 else 1)
        chunk_rows = max(1, min(cfg.m, (2 << 30) // max(per_row, 1)))
    for r0 in range(0, cfg.m, chunk_rows):
        r1 = min(cfg.m, r0 + chunk_rows)
        tt = torch.from_numpy(t[r0:r1]).to(dev)
        ec = torch.exp(-torch.outer(tt, lam_d) * (np.pi ** 2 * cfg.nu)) * coef_d[None, :]
        if cfg.dims == 2:
            T = torch.matmul(ec.view(-1, P, P), Sd[1].t())            # rows x P(p) x gy
            blk = torch.matmul(Sd[0], T)                               # rows x gx x gy
        else:
            T = torch.matmul(ec.view(-1, P * P, P), Sd[2].t())        # rows x (p,q) x gz
            T = T.view(-1, P, P, cfg.grid[2])
            T = torch.einsum("yq,rpqz->rpyz", Sd[1], T)                # rows x P x gy x gz
            blk = torch.einsum("xp,rpyz->rxyz", Sd[0], T)              # rows x gx x gy x gz
        A[r0:r1] = blk.reshape(r1 - r0, ncols).to(out_dtype)
        del T, blk, ec
    if cfg.noise_std:
        for r0 in range(0, cfg.m, 64):
            r1 = min(cfg.m, r0 + 64)
            noise = rng.standard_normal((r1 - r0, cfg.n)) * cfg.noise_std
            A[r0:r1] += torch.from_numpy(noise).to(dev).to(out_dtype)
    return A


def analytic_singular_values(cfg: FieldConfig) -> np.ndarray:
    """sigma(A) of the noise-free field via DST-I orthogonality.

    Phi^T Phi = ((g+1)/2)^d I on the interior grid, so
    sigma(A) = sigma(E diag(c) * ((g+1)/2)^(d/2)) -- an m x P^d SVD.
    """
    _, lam, coef, _ = mode_tables(cfg)
    t = np.linspace(0.0, 1.0, cfg.m)
    e = np.exp(-np.outer(t, lam) * np.pi ** 2 * cfg.nu) * coef[None, :]
    scale = np.prod([np.sqrt((g + 1) / 2.0) for g in cfg.grid])
    return np.linalg.svd(e * scale, compute_uv=False)


def generate_host_columns(cfg: FieldConfig, rows: int, cols) -> np.ndarray:
    """Rows [0, rows) and the given flattened columns of the noise-free field
    as one FP64 GEMM on the host, A[:rows, cols] = (E diag(c)) Phi[cols]^T.

    A timing sample for the CPU baseline of bench.py (the reference's
    per-block work on a bounded piece of a configuration too large for the
    host): the same field, evaluated in another order, so its bytes differ
    from generate_host / generate_device in the last bits -- never a parity
    input."""
    S, lam, coef, _ = mode_tables(cfg)
    t = np.linspace(0.0, 1.0, cfg.m)[:rows]
    ec = np.exp(-np.outer(t, lam) * np.pi ** 2 * cfg.nu) * coef[None, :]
    cols = np.asarray(cols, dtype=np.int64)
    rest = cols
    coords = []
    for g in reversed(cfg.grid):
        coords.append(rest % g)
        rest = rest // g
    coords = coords[::-1]
    P = cfg.modes
    phi = np.ones((cols.size, 1))
    for d, ix in enumerate(coords):
        phi = (phi[:, :, None] * S[d][ix][:, None, :]).reshape(cols.size, -1)
    out = ec @ phi.T
    if cfg.dtype == "f32":
        out = out.astype(np.float32)
    return out
