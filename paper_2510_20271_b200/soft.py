"""Differentiable (soft) ECC with one learnable direction -- ecckit/soft.py on the GPU.

Reference-compatible functions (soft.py:41-257): ``SoftEccParams``,
``SoftGradients``, ``pixel_coordinates``, ``effective_field``,
``reparametrize_direction[_jvp]``, ``soft_ecc``, ``soft_ecc_backward``.

PyTorch surface (the north star's module): ``SoftECCFunction`` (autograd)
and ``SoftECC`` (nn.Module with learnable thresholds tau, direction v -> u =
v/|v| and scale alpha; sharpness lambda is a buffer).  The kernels return
the raw direction gradient -alpha*G; autograd through u = v/|v| supplies the
tangent projection and 1/|v|, i.e. reparametrize_direction_jvp (soft.py:113-121).

Numerics: the reference evaluates in float64.  The engine evaluates the
sigmoid arguments in float32 around a centre m (fp32 accumulation within a
lane, fp64 across lanes and CTAs, fixed order), and the coefficients of the
effective field from a float64 field with the reference's rounding sequence.
Parity contract: normwise relative error <= 1e-4 (max|a-b| / max|b|).
"""

from __future__ import annotations

import functools
import math
from typing import Optional
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .coefficients import CoefficientGrid
from .grid import EulerCurve, ScalarGrid, ThresholdSet

UNIT_NORM_TOL = 1e-12
_LOG2E = 1.4426950408889634
_FACTOR_LIMIT = 40.0  # |log2 a_j| bound for the factorised sigmoid (ecc_soft.cu A_MAX)
_TT = 32  # thresholds per kernel lane


@dataclass(frozen=True)
class SoftEccParams:
    """Sharpness, direction scale, unit direction and thresholds (soft.py:41-63)."""

    lam: float
    alpha: float
    u: np.ndarray
    taus: ThresholdSet

    def __post_init__(self):
        if not self.lam > 0:
            raise ValueError(f"sharpness must be positive, got {self.lam}")
        u = np.asarray(self.u, dtype=np.float64).ravel()
        if u.size not in (2, 3):
            raise ValueError(f"direction must have 2 or 3 components, got {u.size}")
        if not np.isfinite(u).all():
            raise ValueError("direction must be finite")
        if abs(np.linalg.norm(u) - 1.0) > UNIT_NORM_TOL:
            raise ValueError(
                f"direction must be unit length within {UNIT_NORM_TOL}, "
                f"got norm {np.linalg.norm(u)!r}"
            )
        object.__setattr__(self, "u", u)


@dataclass(frozen=True)
class SoftGradients:
    """Cotangent-weighted gradients (soft.py:66-76), plus d_alpha (north star)."""

    d_values: np.ndarray
    d_tau: np.ndarray
    d_u: np.ndarray
    d_alpha: float = field(default=float("nan"))


def pixel_coordinates(dims, start: int = 0, stop: int | None = None) -> np.ndarray:
    """Positions of pixels [start, stop) mapped per axis into [-1, 1] (soft.py:79-94)."""
    dims = tuple(dims)
    n = 1
    for d in dims:
        n *= d
    if stop is None:
        stop = n
    coords = np.unravel_index(np.arange(start, stop), dims)
    out = np.empty((stop - start, len(dims)))
    for a, (idx, d) in enumerate(zip(coords, dims)):
        out[:, a] = 0.0 if d == 1 else idx * (2.0 / (d - 1)) - 1.0
    return out


def reparametrize_direction(v) -> np.ndarray:
    """Map an unconstrained vector onto the unit sphere (soft.py:104-110)."""
    v = np.asarray(v, dtype=np.float64).ravel()
    norm = float(np.linalg.norm(v))
    if norm <= 1e-12:
        raise ValueError(f"direction vector too close to zero (norm {norm!r})")
    return v / norm


def reparametrize_direction_jvp(v, dv) -> np.ndarray:
    """Jacobian-vector product of :func:`reparametrize_direction` (soft.py:113-121)."""
    v = np.asarray(v, dtype=np.float64).ravel()
    dv = np.asarray(dv, dtype=np.float64).ravel()
    norm = float(np.linalg.norm(v))
    if norm <= 1e-12:
        raise ValueError(f"direction vector too close to zero (norm {norm!r})")
    u = v / norm
    return (dv - u * (u @ dv)) / norm


# ---------------------------------------------------------------------------
# device plumbing
# ---------------------------------------------------------------------------

def _soft_tensor(x: torch.Tensor) -> torch.Tensor:
    if x.dtype not in (torch.float32, torch.float64):
        x = x.to(torch.float32)
    return x.contiguous()


def _block_halfwidth(taus) -> float:
    """Largest half-width of the 32-threshold blocks a kernel lane holds."""
    if isinstance(taus, torch.Tensor):
        t = taus.detach().to(torch.float64)
        nb = t.numel()
        pad = (-nb) % _TT
        if pad:
            t = torch.cat([t, t[-1:].expand(pad)])
        blocks = t.reshape(-1, _TT)
        return float(((blocks.max(1).values - blocks.min(1).values) * 0.5).max())
    t = np.asarray(taus, dtype=np.float64)
    return max(0.5 * float(t[i:i + _TT].max() - t[i:i + _TT].min()) for i in range(0, t.size, _TT))


# windowed ("band") kernels, ecc_soft.cu band_ok: 16-threshold blocks, an
# 8-block window per voxel, at most 16 bands, saturation cut 24 ln 2
_BAND_T, _BAND_NWB, _BAND_MAXB, _BAND_MAXBANDS = 16, 8, 368, 16
_BAND_ZCUT = 24.0 * math.log(2.0)


def band_window(taus, lam: float) -> int:
    """Thresholds the soft kernels evaluate per voxel: the 128-threshold window
    of the band kernels when their condition holds (sorted thresholds, every 7
    blocks spanning more than 2 * 24 ln 2 / lam, factorised mode; the device
    decides the same way), else all of them.  For reporting (bench.py)."""
    t = np.asarray(taus.detach().cpu() if isinstance(taus, torch.Tensor) else taus, dtype=np.float64).ravel()
    nb = t.size
    nblk = -(-nb // _BAND_T)
    nbands = nblk - _BAND_NWB + 1
    if nb > _BAND_MAXB or nbands < 2 or nbands > _BAND_MAXBANDS or not np.all(t[:-1] <= t[1:]):
        return nb
    if lam * _LOG2E * _block_halfwidth(t) > _FACTOR_LIMIT:
        return nb
    w2 = 2.0 * _BAND_ZCUT / lam * (1.0 + 1e-3)
    for b in range(nbands - 1):
        if not t[(b + _BAND_NWB) * _BAND_T] - t[(b + 1) * _BAND_T] > w2:
            return nb
    return _BAND_NWB * _BAND_T


def _params(lam: float, alpha: float, u, tau_lo: float, tau_hi: float, ndim: int, halfwidth: float | None = None
            ) -> _lib.SoftParams:
    p = _lib.SoftParams()
    p.lam = float(lam)
    p.alpha = float(alpha)
    uu = np.zeros(3)
    uu[:ndim] = np.asarray(u, dtype=np.float64).ravel()[:ndim]
    for i in range(3):
        p.u[i] = float(uu[i])
    m = 0.5 * (tau_lo + tau_hi)
    p.center = m
    if halfwidth is None:
        halfwidth = 0.5 * (tau_hi - tau_lo)
    # per-lane-block centring keeps |log2 a_j| <= 40 (ecc_soft.cu A_MAX)
    p.factorized = int(lam * _LOG2E * halfwidth <= _FACTOR_LIMIT)
    return p


def soft_prepare_device(x: torch.Tensor, dims, batch: int, p: _lib.SoftParams):
    """(int8 coefficients of the effective field, centred fp32 field, its fp32
    remainder or None) on device; the remainder is only kept in direct mode."""
    code = _lib.dtype_code(x)
    c = torch.empty(x.shape, dtype=torch.int8, device=x.device)
    fc = torch.empty(x.shape, dtype=torch.float32, device=x.device)
    lo = None if p.factorized else torch.empty(x.shape, dtype=torch.float32, device=x.device)
    d = _lib.dims_arg(dims)
    _lib.check(_lib.lib().ecc_soft_prepare(_lib.ptr(x), code, len(dims), _lib.ptr(d), batch, _lib.ctypes.byref(p),
                                           _lib.ptr(c), _lib.ptr(fc), _lib.ptr(lo), _lib.stream_ptr(x)))
    return c, (fc, lo)


def _workspace(dims, batch: int, nb: int, device) -> torch.Tensor:
    d = _lib.dims_arg(dims)
    nbytes = int(_lib.lib().ecc_soft_workspace_bytes(len(dims), _lib.ptr(d), batch, nb))
    return torch.empty(max(nbytes, 8) // 8 + 1, dtype=torch.float64, device=device)


def soft_forward_device(c, field, dims, batch: int, taus_dev: torch.Tensor, p: _lib.SoftParams) -> torch.Tensor:
    fc, lo = field
    nb = taus_dev.numel()
    chi = torch.empty((batch, nb), dtype=torch.float64, device=fc.device)
    ws = _workspace(dims, batch, nb, fc.device)
    d = _lib.dims_arg(dims)
    _lib.check(_lib.lib().ecc_soft_forward(_lib.ptr(c), _lib.ptr(fc), _lib.ptr(lo), len(dims), _lib.ptr(d), batch,
                                           _lib.ptr(taus_dev), nb, _lib.ctypes.byref(p), _lib.ptr(chi), _lib.ptr(ws),
                                           _lib.stream_ptr(fc)))
    return chi


def soft_backward_device(c, field, dims, batch: int, taus_dev, p, upstream: torch.Tensor):
    """(d_values fp32 like the field, d_tau [N,B] fp64, G [N,ndim] fp64)."""
    fc, lo = field
    nb = taus_dev.numel()
    up = upstream.to(torch.float64).contiguous()
    dX = torch.empty(fc.shape, dtype=torch.float32, device=fc.device)
    dtau = torch.empty((batch, nb), dtype=torch.float64, device=fc.device)
    G = torch.empty((batch, len(dims)), dtype=torch.float64, device=fc.device)
    ws = _workspace(dims, batch, nb, fc.device)
    d = _lib.dims_arg(dims)
    _lib.check(_lib.lib().ecc_soft_backward(_lib.ptr(c), _lib.ptr(fc), _lib.ptr(lo), len(dims), _lib.ptr(d), batch,
                                            _lib.ptr(taus_dev), nb, _lib.ctypes.byref(p), _lib.ptr(up), _lib.ptr(dX),
                                            _lib.ptr(dtau), _lib.ptr(G), _lib.ptr(ws), _lib.stream_ptr(fc)))
    return dX, dtau, G


def effective_field(grid: ScalarGrid, alpha: float, u) -> ScalarGrid:
    """The field X + alpha <u, p> (soft.py:97-101), float64, on the device."""
    x = _soft_tensor(grid.device_tensor())
    u = np.ascontiguousarray(np.asarray(u, dtype=np.float64).ravel())
    if u.size != grid.ndim:
        raise ValueError(f"direction has {u.size} components for a {grid.ndim}D grid")
    out = torch.empty(x.shape, dtype=torch.float64, device=x.device)
    d = _lib.dims_arg(grid.dims)
    _lib.check(_lib.lib().ecc_effective_field(_lib.ptr(x), _lib.dtype_code(x), grid.ndim, _lib.ptr(d), 1,
                                              float(alpha), _lib.ptr(u), _lib.ptr(out), _lib.stream_ptr(x)))
    return ScalarGrid(out)


def _check_shapes(grid: ScalarGrid, coeffs: CoefficientGrid, u: np.ndarray):
    if tuple(coeffs.dims) != tuple(grid.dims):
        raise ValueError(f"coefficient dims {coeffs.dims} != grid dims {grid.dims}")
    if u.size != grid.ndim:
        raise ValueError(f"direction has {u.size} components for a {grid.ndim}D grid")


def _coeff_tensor(coeffs: CoefficientGrid, device) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(coeffs.coeffs, dtype=np.int8)).to(device)


def _prepared(grid, coeffs, params):
    x = _soft_tensor(grid.device_tensor())
    taus = params.taus.taus
    p = _params(params.lam, params.alpha, params.u, float(taus[0]), float(taus[-1]), grid.ndim,
                _block_halfwidth(taus))
    _, field = soft_prepare_device(x, grid.dims, 1, p)
    c = _coeff_tensor(coeffs, x.device)
    taus_dev = torch.from_numpy(np.array(taus, dtype=np.float64)).to(x.device)
    return c, field, taus_dev, p


def soft_ecc(grid: ScalarGrid, coeffs: CoefficientGrid, params: SoftEccParams, workers: int = 1) -> EulerCurve:
    """Smoothed Euler characteristic curve (soft.py:182-196), on the GPU.

    ``coeffs`` is expected to come from the effective field; it is taken as
    given (e.g. the reference's own), exactly like the reference.
    """
    _check_shapes(grid, coeffs, params.u)
    c, field, taus_dev, p = _prepared(grid, coeffs, params)
    chi = soft_forward_device(c, field, grid.dims, 1, taus_dev, p)
    return EulerCurve(params.taus.taus, chi[0].cpu().numpy())


def soft_ecc_backward(grid: ScalarGrid, coeffs: CoefficientGrid, params: SoftEccParams, upstream,
                      workers: int = 1) -> SoftGradients:
    """Cotangent-weighted gradients (soft.py:199-257), on the GPU; also d_alpha."""
    _check_shapes(grid, coeffs, params.u)
    upstream = np.asarray(upstream, dtype=np.float64).ravel()
    ntau = len(params.taus)
    if upstream.size != ntau:
        raise ValueError(f"upstream has {upstream.size} weights for {ntau} thresholds")
    c, field, taus_dev, p = _prepared(grid, coeffs, params)
    up = torch.from_numpy(upstream).to(field[0].device).reshape(1, ntau)
    dX, dtau, G = soft_backward_device(c, field, grid.dims, 1, taus_dev, p, up)
    G = G[0].cpu().numpy()
    u = params.u
    d_u = -params.alpha * G
    d_u = d_u - (d_u @ u) * u
    d_alpha = -float(G @ u)
    return SoftGradients(dX.to(torch.float64).cpu().numpy().reshape(grid.dims), dtau[0].cpu().numpy(), d_u,
                         d_alpha)


def gradient_check(grid: ScalarGrid, params: SoftEccParams, upstream=None, step: float = 1e-4,
                   rtol: float = 1e-4, seed: int = 0, workers: int = 1) -> dict:
    """Analytic backward (the CUDA kernels) against 4th-order central finite
    differences (soft.py:260-359), both on the device.

    Same contract as the reference: coefficients from the effective field,
    held fixed; upstream defaults to U(0.5, 1.5) seeded (soft.py:287-289);
    the direction is probed as a free vector and projected onto the tangent
    space; relative errors |a - fd| / max(|a|, |fd|, 1e-4); ``pass`` at rtol
    with tangency <= 1e-8.  The differences come from a float64 harness
    (ecc_soft_fd) that exploits the loss's separability, so the check runs
    at sizes where the reference's O(N) full forward passes are out of reach.
    Extra keys: ``d_alpha`` / ``fd_alpha`` (not in the reference) and ``normwise`` maxima
    ||a - fd||_inf / ||fd||_inf, the acceptance metric of the fp32 engine.
    """
    ntau = len(params.taus)
    if upstream is None:
        upstream = np.random.default_rng(seed).uniform(0.5, 1.5, size=ntau)
    upstream = np.asarray(upstream, dtype=np.float64).ravel()
    if upstream.size != ntau:
        raise ValueError(f"upstream has {upstream.size} weights for {ntau} thresholds")
    u = params.u
    field = effective_field(grid, params.alpha, u)
    from .coefficients import compute_coefficients

    coeffs = compute_coefficients(field)
    grads = soft_ecc_backward(grid, coeffs, params, upstream, workers)

    f = field.device_tensor()
    dev = f.device
    c = _coeff_tensor(coeffs, dev)
    taus_dev = torch.from_numpy(np.array(params.taus.taus, dtype=np.float64)).to(dev)
    up_dev = torch.from_numpy(upstream).to(dev)
    fd_values = torch.empty(f.numel(), dtype=torch.float64, device=dev)
    fd_tau = torch.empty(ntau, dtype=torch.float64, device=dev)
    fd_dir = torch.empty(grid.ndim + 1, dtype=torch.float64, device=dev)
    d = _lib.dims_arg(grid.dims)
    uh = np.ascontiguousarray(u, dtype=np.float64)
    _lib.check(_lib.lib().ecc_soft_fd(_lib.ptr(f), _lib.ptr(c), grid.ndim, _lib.ptr(d), _lib.ptr(taus_dev), ntau,
                                      _lib.ptr(up_dev), float(params.lam), float(params.alpha), _lib.ptr(uh),
                                      float(step), _lib.ptr(fd_values), _lib.ptr(fd_tau), _lib.ptr(fd_dir),
                                      _lib.stream_ptr(f)))
    fd_v = fd_values.cpu().numpy()
    fd_t = fd_tau.cpu().numpy()
    fd_all = fd_dir.cpu().numpy()
    fd_u = fd_all[:grid.ndim]
    fd_u_proj = fd_u - (fd_u @ u) * u
    fd_alpha = float(fd_all[grid.ndim])

    floor = 1e-4

    def rel(a, b):
        a, b = np.atleast_1d(np.asarray(a, np.float64)), np.atleast_1d(np.asarray(b, np.float64))
        return float((np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)).max())

    def normwise(a, b):
        a, b = np.atleast_1d(np.asarray(a, np.float64)), np.atleast_1d(np.asarray(b, np.float64))
        scale = max(float(np.abs(b).max()), floor)
        return float(np.abs(a - b).max() / scale)

    pairs = {"d_values": (grads.d_values.ravel(), fd_v), "d_tau": (grads.d_tau, fd_t), "d_u": (grads.d_u, fd_u_proj),
             "d_alpha": (grads.d_alpha, fd_alpha)}
    report = {k: rel(a, b) for k, (a, b) in pairs.items()}
    report["tangency"] = float(abs(grads.d_u @ u))
    report["fd_alpha"] = fd_alpha
    report["normwise"] = {k: normwise(a, b) for k, (a, b) in pairs.items()}
    report["pass"] = bool(max(report["d_values"], report["d_tau"], report["d_u"]) <= rtol
                          and report["tangency"] <= 1e-8)
    return report


# ---------------------------------------------------------------------------
# PyTorch autograd surface
# ---------------------------------------------------------------------------

# The module path is sync-free: tau, u and alpha stay on the device, the
# kernel parameters (centre, sigmoid mode) are derived there (ecc_soft_setup),
# so a forward + backward issues no device -> host read and can be captured
# in a CUDA graph.  The kernels are registered as torch.library custom ops
# with fake (meta) implementations, so torch.compile traces through them
# without graph breaks.
_PARAMS_F64 = 7   # sizeof(ecc_soft_params) / 8


def _records_bytes(dims, batch: int) -> int:
    d = _lib.dims_arg(dims)
    return int(_lib.lib().ecc_soft_records_bytes(len(dims), _lib.ptr(d), batch))


@torch.library.custom_op("ecc_b200::soft_ecc_fwd", mutates_args=())
def _soft_fwd_op(x: torch.Tensor, taus: torch.Tensor, u: torch.Tensor, alpha: torch.Tensor, lam: float,
                 ndim: int, keep: bool = False
                 ) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor]:
    """(chi [N, B] f64, coefficients int8, centred field f32, its remainder
    f32, device parameters, band records) of x [N, (D,) H, W].  keep: a
    backward will follow -- the windowed kernels then keep their band-sorted
    records (ecc_soft_records_bytes, ~10 B per voxel) so the backward skips
    its compaction and sort; else the records tensor is empty."""
    from .hard import _split_batch

    if not x.is_cuda:
        raise ValueError("SoftECC takes a CUDA tensor")
    dev = x.device
    xs = _soft_tensor(x)
    batch, dims, _ = _split_batch(xs, ndim)
    taus_d = taus.detach().to(dev, torch.float64).contiguous()
    u_d = u.detach().to(dev, torch.float64).contiguous()
    a_d = alpha.detach().to(dev, torch.float64).reshape(1).contiguous()
    nb = taus_d.numel()
    L = _lib.lib()
    st = _lib.stream_ptr(xs)
    params = torch.empty(_PARAMS_F64, dtype=torch.float64, device=dev)
    _lib.check(L.ecc_soft_setup(_lib.ptr(taus_d), nb, _lib.ptr(u_d), ndim, _lib.ptr(a_d), float(lam),
                                _lib.ptr(params), st))
    c = torch.empty(xs.shape, dtype=torch.int8, device=dev)
    fc = torch.empty(xs.shape, dtype=torch.float32, device=dev)
    lo = torch.empty(xs.shape, dtype=torch.float32, device=dev)
    d = _lib.dims_arg(dims)
    _lib.check(L.ecc_soft_prepare_d(_lib.ptr(xs), _lib.dtype_code(xs), len(dims), _lib.ptr(d), batch,
                                    _lib.ptr(params), _lib.ptr(c), _lib.ptr(fc), _lib.ptr(lo), st))
    chi = torch.empty((batch, nb), dtype=torch.float64, device=dev)
    ws = _workspace(dims, batch, nb, dev)
    recs = torch.empty(_records_bytes(dims, batch) if keep else 0, dtype=torch.uint8, device=dev)
    _lib.check(L.ecc_soft_forward_d(_lib.ptr(c), _lib.ptr(fc), _lib.ptr(lo), len(dims), _lib.ptr(d), batch,
                                    _lib.ptr(taus_d), nb, _lib.ptr(params), _lib.ptr(chi), _lib.ptr(ws),
                                    _lib.ptr(recs) if keep else None, st))
    return chi, c, fc, lo, params, recs


@_soft_fwd_op.register_fake
def _(x, taus, u, alpha, lam, ndim, keep=False):
    from .hard import _split_batch

    batch, dims, _ = _split_batch(x, ndim)
    return (x.new_empty((batch, taus.shape[0]), dtype=torch.float64), x.new_empty(x.shape, dtype=torch.int8),
            x.new_empty(x.shape, dtype=torch.float32), x.new_empty(x.shape, dtype=torch.float32),
            x.new_empty((_PARAMS_F64,), dtype=torch.float64),
            x.new_empty((_records_bytes(dims, batch) if keep else 0,), dtype=torch.uint8))


CHUNK_VOXELS = 4096   # ecc_soft.cu CH: voxels per forward chunk


def _stream_3d_item(xs: torch.Tensor, taus, u, alpha, lam: float, keep: bool, slab: int, upstream=None):
    """The streamed forward (and, with ``upstream`` [1, B], the backward) of
    one 3-D item in host memory xs [1?, D, H, W]: z-slabs of ``slab`` planes
    are copied on a side stream; after each slab the compute stream prepares
    the planes whose successor (their halo) has arrived, runs the forward over
    the units whose voxels are prepared and, with an upstream, their backward
    (a unit's backward needs only its own forward records, not chi).  The
    partial rows are reduced once at the end.  Returns (chi, c, fc, lo,
    params, recs, (dX, dtau, G) or None)."""
    dev = taus.device
    L = _lib.lib()
    D, H, W = xs.shape[-3:]
    dims = (D, H, W)
    taus_d = taus.detach().to(dev, torch.float64).contiguous()
    u_d = u.detach().to(dev, torch.float64).contiguous()
    a_d = alpha.detach().to(dev, torch.float64).reshape(1).contiguous()
    nb = taus_d.numel()
    cur = torch.cuda.current_stream(dev)
    st = _lib.ctypes.c_void_p(cur.cuda_stream)
    params = torch.empty(_PARAMS_F64, dtype=torch.float64, device=dev)
    _lib.check(L.ecc_soft_setup(_lib.ptr(taus_d), nb, _lib.ptr(u_d), 3, _lib.ptr(a_d), float(lam),
                                _lib.ptr(params), st))
    xd = torch.empty(xs.shape, dtype=xs.dtype, device=dev)
    c = torch.empty(xs.shape, dtype=torch.int8, device=dev)
    fc = torch.empty(xs.shape, dtype=torch.float32, device=dev)
    lo = torch.empty(xs.shape, dtype=torch.float32, device=dev)
    chi = torch.empty((1, nb), dtype=torch.float64, device=dev)
    ws = _workspace(dims, 1, nb, dev)
    recs = torch.empty(_records_bytes(dims, 1) if keep else 0, dtype=torch.uint8, device=dev)
    bwd = None
    if upstream is not None:
        up = upstream.to(dev, torch.float64).reshape(1, nb).contiguous()
        bwd = (torch.empty(xs.shape, dtype=torch.float32, device=dev),
               torch.empty((1, nb), dtype=torch.float64, device=dev),
               torch.empty((1, 3), dtype=torch.float64, device=dev))
        ws_b = _workspace(dims, 1, nb, dev)   # the backward's partial rows apart from the forward's
    d = _lib.dims_arg(dims)
    g = (_lib.ctypes.c_int64 * 2)()
    _lib.check(L.ecc_soft_units(3, _lib.ptr(d), 1, _lib.ctypes.byref(g, 0), _lib.ctypes.byref(g, 8)))
    per_unit, units = int(g[0]) * CHUNK_VOXELS, int(g[1])
    xv, dv = xs.reshape(D, H, W), xd.view(D, H, W)
    slab = max(1, int(slab))
    side = torch.cuda.Stream(dev)
    side.wait_stream(cur)   # the device buffer's allocation is ordered before the copies
    ready = []
    with torch.cuda.stream(side):
        for z0 in range(0, D, slab):
            z1 = min(D, z0 + slab)
            dv[z0:z1].copy_(xv[z0:z1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
            ready.append((z1, ev))
    rp = _lib.ptr(recs) if keep else None
    fields = (_lib.ptr(c), _lib.ptr(fc), _lib.ptr(lo), 3, _lib.ptr(d), 1, _lib.ptr(taus_d), nb, _lib.ptr(params))

    def run(u0, u1, finish):
        _lib.check(L.ecc_soft_forward_range_d(*fields, _lib.ptr(chi), _lib.ptr(ws), rp, 0, 0, 1, u0, u1, finish,
                                              st))
        if bwd is not None:
            _lib.check(L.ecc_soft_backward_range_d(*fields, _lib.ptr(up), _lib.ptr(bwd[0]), _lib.ptr(bwd[1]),
                                                   _lib.ptr(bwd[2]), _lib.ptr(ws_b), rp, 0, 0, 1, u0, u1, finish, st))

    prepared, done = 0, 0
    for z1, ev in ready:
        cur.wait_event(ev)
        p_end = D if z1 == D else z1 - 1   # plane z1 - 1 waits for its halo z1
        if p_end > prepared:
            _lib.check(L.ecc_soft_prepare_range_d(_lib.ptr(xd), _lib.dtype_code(xd), 3, _lib.ptr(d), 1,
                                                  _lib.ptr(params), _lib.ptr(c), _lib.ptr(fc), _lib.ptr(lo),
                                                  prepared, p_end, st))
            prepared = p_end
        ready_units = units if prepared == D else (prepared * H * W) // per_unit
        if done < ready_units < units:
            run(done, ready_units, 0)
            done = ready_units
    run(done, units, 1)
    return chi, c, fc, lo, params, recs, bwd


def _stream_batch(xs: torch.Tensor, ndim: int, taus, u, alpha, lam: float, keep: bool, group: int, upstream):
    """The streamed forward + backward of a batch xs [N, (D,) H, W] in host
    memory, item groups of ``group`` copied on a side stream; each group is
    prepared (ecc_soft_prepare_d on the group's items) and its forward and
    backward run (ecc_soft_forward_range_d / ecc_soft_backward_range_d over
    the group's item range, the whole batch's buffers) while the next group
    is copied; the partial rows are reduced once at the end.  Returns (chi
    [N, B], dtau [N, B], G [N, ndim])."""
    dev = taus.device
    L = _lib.lib()
    n = xs.shape[0]
    dims = tuple(xs.shape[1:])
    nvox = math.prod(dims)
    taus_d = taus.detach().to(dev, torch.float64).contiguous()
    u_d = u.detach().to(dev, torch.float64).contiguous()
    a_d = alpha.detach().to(dev, torch.float64).reshape(1).contiguous()
    nb = taus_d.numel()
    cur = torch.cuda.current_stream(dev)
    st = _lib.ctypes.c_void_p(cur.cuda_stream)
    params = torch.empty(_PARAMS_F64, dtype=torch.float64, device=dev)
    _lib.check(L.ecc_soft_setup(_lib.ptr(taus_d), nb, _lib.ptr(u_d), ndim, _lib.ptr(a_d), float(lam),
                                _lib.ptr(params), st))
    xd = torch.empty(xs.shape, dtype=xs.dtype, device=dev)
    c = torch.empty(xs.shape, dtype=torch.int8, device=dev)
    fc = torch.empty(xs.shape, dtype=torch.float32, device=dev)
    lo = torch.empty(xs.shape, dtype=torch.float32, device=dev)
    chi = torch.empty((n, nb), dtype=torch.float64, device=dev)
    dX = torch.empty(xs.shape, dtype=torch.float32, device=dev)
    dtau = torch.empty((n, nb), dtype=torch.float64, device=dev)
    G = torch.empty((n, ndim), dtype=torch.float64, device=dev)
    ws, ws_b = _workspace(dims, n, nb, dev), _workspace(dims, n, nb, dev)
    recs = torch.empty(_records_bytes(dims, n) if keep else 0, dtype=torch.uint8, device=dev)
    rp = _lib.ptr(recs) if keep else None
    up = upstream.to(dev, torch.float64).reshape(n, nb).contiguous()
    d = _lib.dims_arg(dims)
    group = max(1, int(group))
    # units sized for one group's launch (a group alone must fill the GPU);
    # the same split on every call of the pass
    g = (_lib.ctypes.c_int64 * 2)()
    _lib.check(L.ecc_soft_units(ndim, _lib.ptr(d), min(group, n), _lib.ctypes.byref(g, 0),
                                _lib.ctypes.byref(g, 8)))
    gcu, units = int(g[0]), int(g[1])
    side = torch.cuda.Stream(dev)
    side.wait_stream(cur)
    ready = []
    with torch.cuda.stream(side):
        for i0 in range(0, n, group):
            i1 = min(n, i0 + group)
            xd[i0:i1].copy_(xs[i0:i1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
            ready.append((i0, i1, ev))
    fields = (_lib.ptr(c), _lib.ptr(fc), _lib.ptr(lo), ndim, _lib.ptr(d), n, _lib.ptr(taus_d), nb, _lib.ptr(params))
    bw = (_lib.ptr(up), _lib.ptr(dX), _lib.ptr(dtau), _lib.ptr(G), _lib.ptr(ws_b), rp)
    for i0, i1, ev in ready:
        cur.wait_event(ev)
        _lib.check(L.ecc_soft_prepare_d(_lib.ptr(xd[i0]), _lib.dtype_code(xd), ndim, _lib.ptr(d), i1 - i0,
                                        _lib.ptr(params), _lib.ptr(c[i0]), _lib.ptr(fc[i0]), _lib.ptr(lo[i0]), st))
        _lib.check(L.ecc_soft_forward_range_d(*fields, _lib.ptr(chi), _lib.ptr(ws), rp, gcu, i0, i1, 0, units, 0,
                                              st))
        _lib.check(L.ecc_soft_backward_range_d(*fields, *bw, gcu, i0, i1, 0, units, 0, st))
    _lib.check(L.ecc_soft_forward_range_d(*fields, _lib.ptr(chi), _lib.ptr(ws), rp, gcu, n, n, 0, units, 1, st))
    _lib.check(L.ecc_soft_backward_range_d(*fields, *bw, gcu, n, n, 0, units, 1, st))
    return chi, dtau, G


def _accumulate_param_grads(module, u, dtau, G) -> None:
    """The parameter gradients SoftECCFunction's backward gives for (d_tau, G)
    of a batch: d_tau summed over items, d_u = -alpha sum G (then autograd
    through u = v/|v|), d_alpha = -<sum G, u>; accumulated into .grad."""
    Gs = G.sum(0)
    outs, grads = [], []
    if module.taus.requires_grad:
        outs.append(module.taus)
        grads.append(dtau.sum(0).to(module.taus.dtype))
    if module.v.requires_grad:
        outs.append(module.direction())
        grads.append((-module.alpha.detach().to(torch.float64) * Gs).to(module.v.dtype))
    if module.alpha.requires_grad:
        outs.append(module.alpha)
        grads.append((-(Gs * u.to(torch.float64)).sum()).to(module.alpha.dtype))
    if outs:
        torch.autograd.backward(outs, grads)


@torch.library.custom_op("ecc_b200::soft_ecc_fwd_host", mutates_args=())
def _soft_fwd_host_op(x_host: torch.Tensor, taus: torch.Tensor, u: torch.Tensor, alpha: torch.Tensor, lam: float,
                      ndim: int, keep: bool = False, slab: int = 64
                      ) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor]:
    """soft_ecc_fwd of one 3-D item held in (pinned) host memory, streamed in
    z-slabs (``_stream_3d_item``): the prepare and the forward of the planes
    already resident overlap the rest of the copy.  The outputs are
    soft_ecc_fwd's for the copied item (the same kernels on the same voxels).
    Other shapes are copied whole and take soft_ecc_fwd."""
    from .hard import _split_batch

    if x_host.is_cuda:
        raise ValueError("soft_ecc_fwd_host takes a host tensor")
    dev = taus.device
    if dev.type != "cuda":
        raise ValueError("the thresholds must be on the CUDA device the item is streamed to")
    xs = _soft_tensor(x_host)
    batch, dims, _ = _split_batch(xs, ndim)
    if ndim != 3 or batch != 1 or not hasattr(_lib.lib(), "ecc_soft_backward_range_d"):
        return _soft_fwd_op(xs.to(dev, non_blocking=True), taus, u, alpha, lam, ndim, keep)
    chi, c, fc, lo, params, recs, _ = _stream_3d_item(xs, taus, u, alpha, lam, keep, slab)
    return chi, c, fc, lo, params, recs


@_soft_fwd_host_op.register_fake
def _(x_host, taus, u, alpha, lam, ndim, keep=False, slab=64):
    from .hard import _split_batch

    batch, dims, _ = _split_batch(x_host, ndim)
    dev = taus.device
    return (torch.empty((batch, taus.shape[0]), dtype=torch.float64, device=dev),
            torch.empty(x_host.shape, dtype=torch.int8, device=dev),
            torch.empty(x_host.shape, dtype=torch.float32, device=dev),
            torch.empty(x_host.shape, dtype=torch.float32, device=dev),
            torch.empty((_PARAMS_F64,), dtype=torch.float64, device=dev),
            torch.empty((_records_bytes(dims, batch) if keep else 0,), dtype=torch.uint8, device=dev))


@torch.library.custom_op("ecc_b200::soft_ecc_bwd", mutates_args=())
def _soft_bwd_op(c: torch.Tensor, fc: torch.Tensor, lo: torch.Tensor, params: torch.Tensor, taus: torch.Tensor,
                 grad_chi: torch.Tensor, ndim: int, recs: Optional[torch.Tensor] = None
                 ) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """(d_values f32 like the field, d_tau [N, B] f64, G [N, ndim] f64) for upstream grad_chi [N, B]."""
    dims = tuple(c.shape[-ndim:])
    batch = c.numel() // math.prod(dims)
    dev = c.device
    taus_d = taus.detach().to(dev, torch.float64).contiguous()
    nb = taus_d.numel()
    up = grad_chi.to(dev, torch.float64).reshape(batch, nb).contiguous()
    dX = torch.empty(fc.shape, dtype=torch.float32, device=dev)
    dtau = torch.empty((batch, nb), dtype=torch.float64, device=dev)
    G = torch.empty((batch, ndim), dtype=torch.float64, device=dev)
    ws = _workspace(dims, batch, nb, dev)
    d = _lib.dims_arg(dims)
    rp = _lib.ptr(recs) if recs is not None and recs.numel() > 0 else None
    _lib.check(_lib.lib().ecc_soft_backward_d(_lib.ptr(c), _lib.ptr(fc), _lib.ptr(lo), ndim, _lib.ptr(d), batch,
                                              _lib.ptr(taus_d), nb, _lib.ptr(params), _lib.ptr(up), _lib.ptr(dX),
                                              _lib.ptr(dtau), _lib.ptr(G), _lib.ptr(ws), rp, _lib.stream_ptr(fc)))
    return dX, dtau, G


@_soft_bwd_op.register_fake
def _(c, fc, lo, params, taus, grad_chi, ndim, recs=None):
    batch = grad_chi.shape[0]
    return (fc.new_empty(fc.shape), fc.new_empty((batch, taus.shape[0]), dtype=torch.float64),
            fc.new_empty((batch, ndim), dtype=torch.float64))


def _soft_setup_context(ctx, inputs, output):
    x, taus, u, alpha, lam, ndim, keep = inputs
    chi, c, fc, lo, params, recs = output
    # the prepared tensors are saved state, not differentiable outputs: no
    # zero gradients are materialised for them (~9 B per voxel of fills)
    ctx.mark_non_differentiable(c, fc, lo, params, recs)
    ctx.set_materialize_grads(False)
    ctx.save_for_backward(c, fc, lo, params, taus, u, alpha, recs)
    ctx.ndim = ndim
    ctx.xdtype = x.dtype


def _soft_backward(ctx, grad_chi, _gc, _gfc, _glo, _gp, _gr):
    c, fc, lo, params, taus, u, alpha, recs = ctx.saved_tensors
    if grad_chi is None:
        return None, None, None, None, None, None, None
    dX, dtau, G = torch.ops.ecc_b200.soft_ecc_bwd(c, fc, lo, params, taus, grad_chi, ctx.ndim, recs)
    Gs = G.sum(0)
    u64 = u.to(Gs.device, torch.float64)
    gx = dX.to(ctx.xdtype) if ctx.needs_input_grad[0] else None
    gt = dtau.sum(0).to(taus.device, taus.dtype) if ctx.needs_input_grad[1] else None
    gu = (-alpha.to(Gs.device, torch.float64) * Gs).to(u.device, u.dtype) if ctx.needs_input_grad[2] else None
    ga = (-(Gs * u64).sum()).to(alpha.device, alpha.dtype) if ctx.needs_input_grad[3] else None
    return gx, gt, gu, ga, None, None, None


torch.library.register_autograd("ecc_b200::soft_ecc_fwd", _soft_backward, setup_context=_soft_setup_context)


def _soft_host_setup_context(ctx, inputs, output):
    _soft_setup_context(ctx, inputs[:7], output)


def _soft_host_backward(ctx, *grads):
    g = _soft_backward(ctx, *grads)
    return (None,) + tuple(g[1:]) + (None,)   # no gradient for the host item; none for slab


torch.library.register_autograd("ecc_b200::soft_ecc_fwd_host", _soft_host_backward,
                                setup_context=_soft_host_setup_context)


@functools.lru_cache(maxsize=None)
def _total_memory_idx(index: int) -> int:
    return int(torch.cuda.get_device_properties(index).total_memory)


def _total_memory(device: torch.device) -> int:
    return _total_memory_idx(device.index if device.index is not None else torch.cuda.current_device())


class SoftECCFunction:
    """chi[N, B] = sum_p c_p sigmoid(lam (tau_j - X_np - alpha <u, pos_p>)).

    x: CUDA [N, (D,) H, W] float32/float64; taus: [B]; u: [ndim] (any norm;
    the module normalises); alpha: scalar tensor; lam: python float.
    Coefficients come from the effective field and carry no gradient
    (soft.py:14-19).  Differentiable in x, taus, u and alpha
    through the registered custom op ``torch.ops.ecc_b200.soft_ecc_fwd``.
    """

    # band records are kept for the backward while they stay below this
    # fraction of the device's memory (~10 B per voxel on top of the 9 B of
    # saved coefficients and field); above it the backward re-sorts instead
    RECORDS_MEMORY_FRACTION = 0.125

    @staticmethod
    def apply(x, taus, u, alpha, lam: float, ndim: int):
        keep = torch.is_grad_enabled() and any(t.requires_grad for t in (x, taus, u, alpha))
        if keep and x.is_cuda:
            cap = _total_memory(x.device) * SoftECCFunction.RECORDS_MEMORY_FRACTION
            keep = 10 * x.numel() <= cap
        chi = torch.ops.ecc_b200.soft_ecc_fwd(x, taus, u, alpha, float(lam), int(ndim), keep)[0]
        return chi if x.dim() == ndim + 1 else chi[0]


class SoftECC(torch.nn.Module):
    """Single-direction differentiable ECC layer (the paper's PyTorch module).

    Learnable: thresholds ``taus`` [B], direction ``v`` [ndim] (u = v/|v|,
    soft.py:104-110), scale ``alpha``.  Buffer: sharpness ``lam``.
    forward(x [N?, (D,) H, W]) -> chi [N?, B] (float64).
    """

    def __init__(self, taus, direction, alpha: float = 0.0, lam: float = 50.0, ndim: int | None = None,
                 learn_taus: bool = True, learn_direction: bool = True, learn_alpha: bool = True):
        super().__init__()
        taus = torch.as_tensor(np.asarray(taus, dtype=np.float64))
        v = torch.as_tensor(np.asarray(direction, dtype=np.float64).ravel())
        if v.numel() not in (2, 3):
            raise ValueError(f"direction must have 2 or 3 components, got {v.numel()}")
        if float(v.norm()) <= 1e-12:
            raise ValueError("direction vector too close to zero")
        if not lam > 0:
            raise ValueError(f"sharpness must be positive, got {lam}")
        self.ndim = int(v.numel()) if ndim is None else int(ndim)
        self.taus = torch.nn.Parameter(taus, requires_grad=learn_taus)
        self.v = torch.nn.Parameter(v, requires_grad=learn_direction)
        self.alpha = torch.nn.Parameter(torch.tensor(float(alpha), dtype=torch.float64), requires_grad=learn_alpha)
        self.register_buffer("lam", torch.tensor(float(lam), dtype=torch.float64))
        self._lam = float(lam)   # the kernels take lambda by value: no device read per call

    def direction(self) -> torch.Tensor:
        return self.v / self.v.norm()

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return SoftECCFunction.apply(x, self.taus, self.direction(), self.alpha, self._lam, self.ndim)


def soft_step_host(module: SoftECC, host_x: torch.Tensor, upstream: torch.Tensor | None = None,
                   micro: int = 4, slab_planes: int = 16) -> torch.Tensor:
    """Forward + backward of ``module`` on a batch held in (pinned) host
    memory, with the host -> device copies overlapped with the compute.

    The items go to the device in groups of ``micro`` on a side stream; as
    each group arrives its prepare, forward and backward run (the upstream is
    given, so no item waits for another's chi) over the whole batch's
    buffers, and the partial rows are reduced once at the end
    (``_stream_batch``).  A single 3-D item ([1, D, H, W]) is streamed in
    z-slabs of ``slab_planes`` planes instead (``_stream_3d_item``).  Either
    way chi and the parameter gradients (accumulated into ``.grad``) are the
    device path's, bit for bit.  Without gradients (or an older library) the
    batch runs in micro-batches of ``micro`` items through the module, the
    next one copied while the current one computes.
    upstream: d loss / d chi [N, B] (default ones).  Returns chi [N, B] on
    the device (enqueued; nothing here synchronises the host).
    """
    if host_x.is_cuda:
        raise ValueError("soft_step_host takes a host tensor (pin it for asynchronous copies)")
    dev = module.taus.device
    n = host_x.shape[0]
    if module.ndim == 3 and host_x.dim() == 4 and n == 1 and dev.type == "cuda":
        # one 3-D item: streamed in z-slabs, the prepare and the forward of the
        # resident planes overlapping the rest of the copy
        # resident planes, and -- the upstream being given -- the backward of
        # each unit right after its forward; the parameter gradients are those
        # of SoftECCFunction's backward (soft_ecc_bwd + autograd through u = v/|v|)
        params = [t for t in (module.taus, module.v, module.alpha) if t.requires_grad]
        grad = torch.is_grad_enabled() and bool(params)
        keep = grad and 10 * host_x.numel() <= _total_memory(dev) * SoftECCFunction.RECORDS_MEMORY_FRACTION
        up = None
        if grad:
            nb = module.taus.numel()
            up = (torch.ones((1, nb), dtype=torch.float64, device=dev) if upstream is None
                  else upstream.to(dev, torch.float64, non_blocking=True).reshape(1, nb))
        with torch.no_grad():
            u = module.direction()
            chi, *_, bwd = _stream_3d_item(_soft_tensor(host_x), module.taus, u, module.alpha, module._lam,
                                           keep, slab_planes, up)
        if grad:
            _accumulate_param_grads(module, u, bwd[1], bwd[2])
        return chi
    params = [t for t in (module.taus, module.v, module.alpha) if t.requires_grad]
    if (torch.is_grad_enabled() and params and dev.type == "cuda" and host_x.dim() == module.ndim + 1
            and hasattr(_lib.lib(), "ecc_soft_backward_range_d")):
        # a batch: item groups streamed, each group's prepare, forward and
        # backward overlapping the next group's copy (one reduction at the end)
        nb = module.taus.numel()
        up = (torch.ones((n, nb), dtype=torch.float64, device=dev) if upstream is None
              else upstream.to(dev, torch.float64, non_blocking=True).reshape(n, nb))
        keep = 10 * host_x.numel() <= _total_memory(dev) * SoftECCFunction.RECORDS_MEMORY_FRACTION
        with torch.no_grad():
            u = module.direction()
            chi, dtau, G = _stream_batch(_soft_tensor(host_x), module.ndim, module.taus, u, module.alpha,
                                         module._lam, keep, micro, up)
        _accumulate_param_grads(module, u, dtau, G)
        return chi
    micro = max(1, min(int(micro), n))
    cur = torch.cuda.current_stream(dev)
    side = torch.cuda.Stream(dev)
    bufs = [torch.empty((micro,) + tuple(host_x.shape[1:]), dtype=host_x.dtype, device=dev) for _ in range(2)]
    freed = [None, None]
    chis = []
    for k, i0 in enumerate(range(0, n, micro)):
        i1 = min(n, i0 + micro)
        buf = bufs[k % 2][: i1 - i0]
        with torch.cuda.stream(side):
            if freed[k % 2] is not None:
                side.wait_event(freed[k % 2])
            buf.copy_(host_x[i0:i1], non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(side)
        cur.wait_event(ready)
        buf.record_stream(cur)
        chi = module(buf)
        if chi.requires_grad:   # forward only without gradients
            up = torch.ones_like(chi) if upstream is None else upstream[i0:i1].to(dev, chi.dtype, non_blocking=True)
            chi.backward(up)
        chis.append(chi.detach())
        done = torch.cuda.Event()
        done.record(cur)
        freed[k % 2] = done
    return torch.cat(chis)
