"""Seeded synthetic inputs for the five BASELINE.json configurations.

Input generation only (see package docstring): every function here returns
coordinates or field VALUES evaluated from closed-form synthetic recipes.  The
recipes (documented in DESIGN.md "Input recipe") stand in for the paper's MAS
coronal relaxation run (Sec. 5, Table 1), which cannot be reproduced:
  * geometrically stretched r grid, uniform theta / phi (Table 1 shape),
  * tilted-dipole / multipole unit field b (Sec. 5 "potential solution"),
  * 1-2 MK corona with a transition-region ramp (Sec. 4.1, Fig. 5),
  * density falling as r^-4 for the viscosity coefficient nu*rho (Sec. 4.1).

Storage convention shared with both implementations (an interface, not
arithmetic): every field is a C-contiguous float64 array of shape (n1, n2, n3)
with n3 (phi / z) fastest.  Face fields use the "+ face" convention:
f1[i,j,k] lives on face (i+1/2, j, k), f2[i,j,k] on (i, j+1/2, k), f3[i,j,k] on
(i, j, k+1/2) (for periodic dim 3, f3[..., n3-1] is the wrap face).
Vector fields with ncomp components are stacked as (ncomp, n1, n2, n3).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

__all__ = [
    "Grid", "uniform_cartesian", "spherical_grid", "geometric_faces", "subgrid", "r_slab", "split_planes",
    "gaussian_bump", "tilted_dipole_b", "multipole_b", "smooth_modes",
    "corona_T", "tr_corona_T", "viscosity_inputs", "constant_faces",
    "CONFIGS", "SPITZER", "make_config", "cartesian_mesh", "random_unit_b",
]


@dataclass
class Grid:
    """Logically rectangular tensor-product grid (Sec. 4.2, Table 1)."""
    geom: str                 # "cartesian" or "spherical" (r, theta, phi)
    x1f: np.ndarray           # n1+1 face coordinates (r or x)
    x2f: np.ndarray           # n2+1 face coordinates (theta or y)
    x3f: np.ndarray           # n3+1 face coordinates (phi or z)
    periodic3: bool = False   # dim-3 periodic (phi)
    x1c: np.ndarray = field(default=None)
    x2c: np.ndarray = field(default=None)
    x3c: np.ndarray = field(default=None)
    x1_span: tuple = None      # (x1 min, x1 max) of the GLOBAL grid when this is an r-slab

    def __post_init__(self):
        self.x1f = np.ascontiguousarray(self.x1f, dtype=np.float64)
        self.x2f = np.ascontiguousarray(self.x2f, dtype=np.float64)
        self.x3f = np.ascontiguousarray(self.x3f, dtype=np.float64)
        # cell centres are part of the grid definition: face midpoints
        if self.x1c is None:
            self.x1c = 0.5 * (self.x1f[1:] + self.x1f[:-1])
        if self.x2c is None:
            self.x2c = 0.5 * (self.x2f[1:] + self.x2f[:-1])
        if self.x3c is None:
            self.x3c = 0.5 * (self.x3f[1:] + self.x3f[:-1])

    @property
    def span1(self):
        return self.x1_span if self.x1_span is not None else (float(self.x1f[0]), float(self.x1f[-1]))

    @property
    def shape(self):
        return (len(self.x1f) - 1, len(self.x2f) - 1, len(self.x3f) - 1)

    @property
    def ncells(self):
        n1, n2, n3 = self.shape
        return n1 * n2 * n3

    @property
    def period3(self) -> float:
        return float(self.x3f[-1] - self.x3f[0]) if self.periodic3 else 0.0


def uniform_cartesian(n1, n2, n3, h=1.0) -> Grid:
    """Config 0: uniform Cartesian box, spacing h, zero-flux walls."""
    return Grid("cartesian", np.arange(n1 + 1) * h, np.arange(n2 + 1) * h,
                np.arange(n3 + 1) * h, periodic3=False)


def geometric_faces(x0: float, x1: float, n: int, first: float) -> np.ndarray:
    """n cells on [x0, x1] whose widths grow geometrically from `first`.

    The stretch ratio q solves first*(q^n - 1)/(q - 1) = x1 - x0 (bisection).
    """
    length = x1 - x0
    if n * first >= length:  # uniform (or compressive) fallback
        return np.linspace(x0, x1, n + 1)

    def total(q):
        return first * n if abs(q - 1.0) < 1e-15 else first * (q ** n - 1.0) / (q - 1.0)

    lo, hi = 1.0, 2.0
    while total(hi) < length:
        hi *= 2.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if total(mid) < length:
            lo = mid
        else:
            hi = mid
    q = 0.5 * (lo + hi)
    widths = first * q ** np.arange(n)
    faces = x0 + np.concatenate([[0.0], np.cumsum(widths)])
    faces[-1] = x1
    return faces


def spherical_grid(nr, nt, nphi, r0=1.0, r1=20.0, dr0=0.005) -> Grid:
    """Configs 1-4: r geometric from r0 (first cell dr0), theta in (0, pi), phi periodic."""
    return Grid("spherical", geometric_faces(r0, r1, nr, dr0),
                np.linspace(0.0, math.pi, nt + 1),
                np.linspace(0.0, 2.0 * math.pi, nphi + 1), periodic3=True)


def r_slab(grid: Grid, i0: int, nl: int) -> Grid:
    """The r-planes [i0, i0+nl) of `grid` (fields evaluated on it equal the
    corresponding planes of the global fields)."""
    return Grid(grid.geom, grid.x1f[i0:i0 + nl + 1], grid.x2f, grid.x3f, periodic3=grid.periodic3,
                x1c=grid.x1c[i0:i0 + nl], x2c=grid.x2c, x3c=grid.x3c, x1_span=grid.span1)


def split_planes(n1: int, nparts: int):
    """Balanced contiguous split of n1 planes: [(i0, nl)] (sizes differ by <= 1)."""
    base, rem = divmod(n1, nparts)
    out, i0 = [], 0
    for p in range(nparts):
        nl = base + (1 if p < rem else 0)
        out.append((i0, nl))
        i0 += nl
    return out


def subgrid(grid: Grid, c, radius: int):
    """Index box of half-width `radius` around cell c=(i,j,k).

    Returns (sub_grid, (I, J, K) index arrays into the parent, local index of c).
    Dims 1/2 are clipped at the physical boundary (so a box touching it keeps the
    true boundary); periodic dim 3 wraps with unwrapped coordinates.  Used by the
    full-size sampled parity tests to evaluate the oracle on a neighbourhood.
    """
    n1, n2, n3 = grid.shape
    i, j, k = c
    I = np.arange(max(0, i - radius), min(n1, i + radius + 1))
    J = np.arange(max(0, j - radius), min(n2, j + radius + 1))
    if grid.periodic3 and n3 > 2 * radius + 1:
        K = np.arange(k - radius, k + radius + 1)
        shift = np.floor_divide(K, n3)
        Kw = K - shift * n3
        x3c = grid.x3c[Kw] + shift * grid.period3
        x3f = np.concatenate([[grid.x3f[Kw[0]] + shift[0] * grid.period3],
                              grid.x3f[Kw + 1] + shift * grid.period3])
        per = False
        kloc = radius
    elif grid.periodic3:
        Kw = np.arange(n3)
        x3c, x3f, per, kloc = grid.x3c.copy(), grid.x3f.copy(), True, k
    else:
        Kw = np.arange(max(0, k - radius), min(n3, k + radius + 1))
        x3c = grid.x3c[Kw]
        x3f = grid.x3f[Kw[0]:Kw[-1] + 2]
        per, kloc = False, k - Kw[0]
    sub = Grid(grid.geom, grid.x1f[I[0]:I[-1] + 2], grid.x2f[J[0]:J[-1] + 2], x3f,
               periodic3=per, x1c=grid.x1c[I], x2c=grid.x2c[J], x3c=x3c, x1_span=grid.span1)
    return sub, (I, J, Kw), (i - I[0], j - J[0], kloc)


# --------------------------------------------------------------------------
# meshes and fields (torch; evaluated on any device, float64)
# --------------------------------------------------------------------------
def _mesh(grid: Grid, device, which=("c", "c", "c")):
    a = torch.as_tensor(grid.x1c if which[0] == "c" else grid.x1f[1:], dtype=torch.float64, device=device)
    b = torch.as_tensor(grid.x2c if which[1] == "c" else grid.x2f[1:], dtype=torch.float64, device=device)
    c = torch.as_tensor(grid.x3c if which[2] == "c" else grid.x3f[1:], dtype=torch.float64, device=device)
    return a[:, None, None], b[None, :, None], c[None, None, :]


def cartesian_mesh(grid: Grid, device="cpu"):
    """Cartesian coordinates (x, y, z) of cell centres (broadcastable tensors)."""
    r, t, p = _mesh(grid, device)
    if grid.geom == "cartesian":
        return r, t, p
    st = torch.sin(t)
    return r * st * torch.cos(p), r * st * torch.sin(p), r * torch.cos(t) + 0 * p


def constant_faces(grid: Grid, value=1.0, device="cpu"):
    n1, n2, n3 = grid.shape
    f = torch.full((n1, n2, n3), float(value), dtype=torch.float64, device=device)
    return f, f.clone(), f.clone()


def gaussian_bump(grid: Grid, sigma=4.0, noise=1e-3, seed=0, device="cpu"):
    """Config 0 initial u: Gaussian (sigma in length units) at the box centre + U(0,1)*noise."""
    x, y, z = cartesian_mesh(grid, device)
    cx = 0.5 * (grid.x1f[0] + grid.x1f[-1])
    cy = 0.5 * (grid.x2f[0] + grid.x2f[-1])
    cz = 0.5 * (grid.x3f[0] + grid.x3f[-1])
    u = torch.exp(-((x - cx) ** 2 + (y - cy) ** 2 + (z - cz) ** 2) / (2.0 * sigma ** 2))
    rng = np.random.default_rng(seed)
    u = u + noise * torch.as_tensor(rng.random(grid.shape), dtype=torch.float64, device=device)
    return u.contiguous()


def _to_spherical_components(grid, bx, by, bz, device):
    r, t, p = _mesh(grid, device)
    st, ct, sp, cp = torch.sin(t), torch.cos(t), torch.sin(p), torch.cos(p)
    br = bx * st * cp + by * st * sp + bz * ct
    bt = bx * ct * cp + by * ct * sp - bz * st
    bp = -bx * sp + by * cp
    return br, bt, bp


def _dipole(x, y, z, m, x0=(0.0, 0.0, 0.0)):
    dx, dy, dz = x - x0[0], y - x0[1], z - x0[2]
    rr = torch.sqrt(dx * dx + dy * dy + dz * dz)
    mr = (m[0] * dx + m[1] * dy + m[2] * dz) / rr
    inv3 = 1.0 / rr ** 3
    return ((3 * mr * dx / rr - m[0]) * inv3, (3 * mr * dy / rr - m[1]) * inv3,
            (3 * mr * dz / rr - m[2]) * inv3)


def _unit_b_from_cartesian(grid, bx, by, bz, device):
    bx, by, bz = [torch.broadcast_to(v, grid.shape) for v in (bx, by, bz)]
    if grid.geom == "spherical":
        b1, b2, b3 = _to_spherical_components(grid, bx, by, bz, device)
    else:
        b1, b2, b3 = bx, by, bz
    nrm = torch.sqrt(b1 * b1 + b2 * b2 + b3 * b3)
    return torch.stack([b1 / nrm, b2 / nrm, b3 / nrm]).contiguous()


def tilted_dipole_b(grid: Grid, tilt_deg=30.0, device="cpu"):
    """Config 1/2: unit vector of a dipole tilted by tilt_deg from the z axis.

    Returns (3, n1, n2, n3): components along the grid's own unit vectors
    (r, theta, phi for spherical grids).
    """
    a = math.radians(tilt_deg)
    m = (math.sin(a), 0.0, math.cos(a))
    x, y, z = cartesian_mesh(grid, device)
    return _unit_b_from_cartesian(grid, *_dipole(x, y, z, m), device)


def multipole_b(grid: Grid, seed=3, n_extra=6, device="cpu"):
    """Config 3/4: tilted dipole plus random sub-surface dipoles (a multipole field)."""
    rng = np.random.default_rng(seed)
    x, y, z = cartesian_mesh(grid, device)
    a = math.radians(20.0)
    bx, by, bz = _dipole(x, y, z, (math.sin(a), 0.0, math.cos(a)))
    for _ in range(n_extra):
        d = rng.normal(size=3)
        pos = 0.6 * d / np.linalg.norm(d) * rng.uniform(0.3, 1.0)
        m = rng.normal(size=3) * 0.08
        ex, ey, ez = _dipole(x, y, z, tuple(m), tuple(pos))
        bx, by, bz = bx + ex, by + ey, bz + ez
    return _unit_b_from_cartesian(grid, bx, by, bz, device)


def random_unit_b(grid: Grid, seed=0, device="cpu"):
    """Rough per-cell random unit vectors (worst-case data for parity tests only)."""
    rng = np.random.default_rng(seed)
    v = torch.as_tensor(rng.normal(size=(3,) + grid.shape), dtype=torch.float64, device=device)
    return (v / torch.sqrt((v * v).sum(0, keepdim=True))).contiguous()


def smooth_modes(grid: Grid, seed=1, nmodes=8, device="cpu"):
    """Sum of seeded smooth separable modes, normalised so |S| <= 1.

    Radial argument is log-radius (the stretched r grid is uniform in log r),
    angular modes are integer so phi-periodicity holds.
    """
    rng = np.random.default_rng(seed)
    r, t, p = _mesh(grid, device)
    r_lo, r_hi = grid.span1
    if grid.geom == "spherical":
        rho = torch.log(r / r_lo) / math.log(r_hi / r_lo)
        tt, pp = t, p
    else:
        rho = (r - r_lo) / (r_hi - r_lo)
        tt = math.pi * (t - grid.x2f[0]) / (grid.x2f[-1] - grid.x2f[0])
        pp = 2 * math.pi * (p - grid.x3f[0]) / (grid.x3f[-1] - grid.x3f[0])
    amps = rng.uniform(-1, 1, nmodes)
    S = torch.zeros(grid.shape, dtype=torch.float64, device=device)
    for a in amps:
        kp, kt, km = rng.integers(1, 4), rng.integers(1, 5), rng.integers(0, 4)
        ph = rng.uniform(0, 2 * math.pi, 3)
        S = S + a * torch.sin(kp * math.pi * rho + ph[0]) * torch.cos(kt * tt + ph[1]) \
            * torch.cos(km * pp + ph[2])
    return (S / np.abs(amps).sum()).contiguous()


def corona_T(grid: Grid, seed=1, T0=1.5e6, amp=0.3, device="cpu"):
    """Config 1: T = T0 * (1 + amp * S), S seeded smooth modes."""
    return (T0 * (1.0 + amp * smooth_modes(grid, seed, device=device))).contiguous()


def tr_corona_T(grid: Grid, seed=2, T_ch=2.0e4, r_tr=1.01, w_tr=0.002, device="cpu"):
    """Config 3: 1-2 MK corona with a steep transition-region ramp below r = 1.02."""
    r, _, _ = _mesh(grid, device)
    T_cor = 1.5e6 + 0.5e6 * smooth_modes(grid, seed, device=device)
    ramp = 0.5 * (1.0 + torch.tanh((r - r_tr) / w_tr))
    return (T_ch + (T_cor - T_ch) * ramp).contiguous()


def viscosity_inputs(grid: Grid, seed=4, nu=1.0, amp=1e-2, nmodes=6, device="cpu"):
    """Config 2: rho ~ r^-4 at cells, nu*rho evaluated at face positions, and a
    solenoidal velocity v = curl(Psi) (Cartesian components), Psi = sum of seeded
    Fourier modes, scaled so |v| <= amp (sum of the mode amplitudes = amp).

    Returns (rho, (f1, f2, f3), v[3, n1, n2, n3]).
    """
    rng = np.random.default_rng(seed)
    rc, _, _ = _mesh(grid, device)
    rf, _, _ = _mesh(grid, device, which=("f", "c", "c"))
    shape = grid.shape
    rho = torch.broadcast_to(1.0 / ((rc * rc) * (rc * rc)), shape).contiguous()
    f1 = torch.broadcast_to(nu / ((rf * rf) * (rf * rf)), shape).contiguous()
    f2 = torch.broadcast_to(nu / ((rc * rc) * (rc * rc)), shape).contiguous()
    f3 = f2.clone()
    x, y, z = cartesian_mesh(grid, device)
    v = torch.zeros((3,) + shape, dtype=torch.float64, device=device)
    bound = 0.0
    for _ in range(nmodes):
        k = rng.normal(size=3) * 1.5
        c = rng.normal(size=3)
        ph = rng.uniform(0, 2 * math.pi)
        kxc = np.cross(k, c)
        bound += float(np.linalg.norm(kxc))
        arg = torch.cos(k[0] * x + k[1] * y + k[2] * z + ph)
        for d in range(3):
            v[d] += kxc[d] * arg
    v = v * (amp / bound)    # |v| <= amp everywhere; independent of the slab evaluated
    return rho, (f1, f2, f3), v.contiguous()


# --------------------------------------------------------------------------
# BASELINE.json configurations
# --------------------------------------------------------------------------
CONFIGS = {
    # name: (kind, shape, dt_ratio list)
    "c0_heat32": ("heat", (32, 32, 32), (50.0,)),
    "c1_spitzer64": ("spitzer", (64, 64, 128), (100.0,)),
    "c2_visc64": ("visc", (64, 64, 128), (500.0,)),
    "c3_spitzer256": ("spitzer_tr", (256, 256, 512), (10.0, 100.0, 1000.0)),
    "c4_scale512": ("spitzer_tr+visc", (512, 512, 1024), (300.0,)),
}

SPITZER = dict(kappa0=1.0e-9, T_cut=5.0e5)  # kappa0 scale is irrelevant: dt is set in units of dt_exp


def make_config(name: str, device="cpu", shape=None, seed=0, slab=None):
    """Build every input of a BASELINE.json config.  `shape` overrides the size
    (for scaled-down parity runs of the same recipe); `slab=(i0, nl)` builds
    only those r-planes of the global fields (one rank's share)."""
    kind, default_shape, ratios = CONFIGS[name]
    n1, n2, n3 = shape or default_shape
    out = {"name": name, "kind": kind, "dt_ratios": ratios}
    if kind == "heat":
        g = uniform_cartesian(n1, n2, n3, 1.0)
        out.update(grid=g, u=gaussian_bump(g, sigma=4.0, noise=1e-3, seed=seed, device=device),
                   faces=constant_faces(g, 1.0, device), b=None, w=None, mode="iso")
        return out
    g = spherical_grid(n1, n2, n3)
    out["global_grid"] = g
    if slab is not None:
        g = r_slab(g, *slab)
    out["grid"] = g
    if kind == "spitzer":
        out.update(T=corona_T(g, seed=seed + 1, device=device),
                   b=tilted_dipole_b(g, 30.0, device=device), mode="aniso", **SPITZER)
    elif kind in ("spitzer_tr", "spitzer_tr+visc"):
        out.update(T=tr_corona_T(g, seed=seed + 2, device=device),
                   b=multipole_b(g, seed=seed + 3, device=device), mode="aniso", **SPITZER)
    if kind in ("visc", "spitzer_tr+visc"):
        rho, vf, v = viscosity_inputs(g, seed=seed + 4, device=device)
        out.update(rho=rho, visc_faces=vf, v=v)
        if kind == "visc":
            out["mode"] = "iso"
    return out
