"""Grid, coefficient and curve files, and the loader that streams a grid file
into device memory.

File formats are the reference's, byte for byte (ecckit/grid.py:11-21):

    magic "ECCG" | version u8 | ndim u8 in {2,3} | reserved u16 = 0
    | dims as ndim x u64 little-endian
    | payload: prod(dims) x f32 (version 1, grids) or i32 (version 2,
      coefficients), little-endian, row-major

with the same validation order and exception types as grid.py:235-278
(FormatError for the header, CorruptionError for a payload that does not
match it, ValueError from ScalarGrid for non-finite values, OSError for a
missing file), and the curve CSV of grid.py:300-323.

The device side is new: ``load_grid_device`` reads the payload (or a range
of planes along axis 0) through two pinned staging buffers, so the file read
of one chunk overlaps the host-to-device copy of the previous one, and checks
finiteness on the device (the min/max pass the thresholds need anyway).
``load_slab_device`` gives each rank of a z-slab partition its own planes
plus the two neighbour planes straight from the file, which replaces the
halo exchange for file-backed volumes.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from .coefficients import COEFF_RANGE, CoefficientGrid
from .grid import CorruptionError, EulerCurve, FormatError, ScalarGrid

MAGIC = b"ECCG"
VERSION_SCALAR = 1
VERSION_COEFF = 2
_HEADER = struct.Struct("<4sBBH")


@dataclass(frozen=True)
class GridHeader:
    """Parsed header: format version, extents and the payload's byte offset."""

    version: int
    dims: tuple
    offset: int

    @property
    def count(self) -> int:
        n = 1
        for d in self.dims:
            n *= d
        return n


def pack_header(version: int, dims) -> bytes:
    """Header bytes of a grid file (grid.py:233-235)."""
    return _HEADER.pack(MAGIC, version, len(dims), 0) + np.asarray(dims, dtype="<u8").tobytes()


def parse_header(data: bytes, path="<bytes>") -> GridHeader:
    """Validate and parse a header (grid.py:238-256): length, magic, reserved
    field, ndim byte, dims block, zero extents -- in that order."""
    if len(data) < _HEADER.size:
        raise FormatError(f"{path}: {len(data)} bytes, too short for an ECCG header")
    magic, version, ndim, reserved = _HEADER.unpack_from(data)
    if magic != MAGIC:
        raise FormatError(f"{path}: not an ECCG file (magic {magic!r})")
    if reserved != 0:
        raise FormatError(f"{path}: header reserved word must be 0, found {reserved}")
    if ndim not in (2, 3):
        raise FormatError(f"{path}: unsupported dimensionality {ndim} (2 or 3)")
    end = _HEADER.size + 8 * ndim
    if len(data) < end:
        raise FormatError(f"{path}: header ends inside the extents block")
    dims = tuple(int(d) for d in np.frombuffer(data, dtype="<u8", count=ndim, offset=_HEADER.size))
    if any(d == 0 for d in dims):
        raise FormatError(f"{path}: empty extent in {dims}")
    return GridHeader(version, dims, end)


def read_header(path, expected_version: int | None = None, itemsize: int = 4) -> GridHeader:
    """Header of a file on disk, with the version and payload-size checks of
    grid.py:259-277 (without reading the payload)."""
    path = Path(path)
    with open(path, "rb") as f:
        head = f.read(_HEADER.size + 24)
    h = parse_header(head, path)
    if expected_version is not None and h.version != expected_version:
        raise FormatError(f"{path}: format version {h.version}, this reader takes {expected_version}")
    _check_payload(path, h, path.stat().st_size, itemsize)
    return h


def _check_payload(path, h: GridHeader, file_size: int, itemsize: int) -> None:
    want = h.count * itemsize
    if file_size - h.offset != want:
        raise CorruptionError(f"{path}: {file_size - h.offset} payload bytes, extents {h.dims} need {want}")


def _read_payload(path, expected_version: int, dtype: str):
    path = Path(path)
    data = path.read_bytes()
    h = parse_header(data, path)
    if h.version != expected_version:
        raise FormatError(f"{path}: format version {h.version}, this reader takes {expected_version}")
    _check_payload(path, h, len(data), np.dtype(dtype).itemsize)
    return np.frombuffer(data, dtype=dtype, count=h.count, offset=h.offset), h.dims


def read_grid(path) -> ScalarGrid:
    """Read a version-1 grid file (grid.py:280-283)."""
    payload, dims = _read_payload(path, VERSION_SCALAR, "<f4")
    return ScalarGrid(payload.astype(np.float64).reshape(dims))


def write_grid(grid, path) -> None:
    """Write a version-1 grid file with a float32 payload (grid.py:286-295).
    Accepts a ScalarGrid or a (host or device) array/tensor."""
    if isinstance(grid, torch.Tensor):
        values, dims = grid.detach().cpu().numpy(), tuple(grid.shape)
    elif isinstance(grid, ScalarGrid):
        values, dims = grid.values, grid.dims
    else:
        values = np.asarray(grid)
        dims = values.shape
    Path(path).write_bytes(pack_header(VERSION_SCALAR, dims) + np.ascontiguousarray(values).astype("<f4").tobytes())


def write_coefficients(cg: CoefficientGrid, path) -> None:
    """Write a version-2 file with an int32 payload (coefficients.py:183-186)."""
    coeffs = cg.coeffs.detach().cpu().numpy() if isinstance(cg.coeffs, torch.Tensor) else np.asarray(cg.coeffs)
    Path(path).write_bytes(pack_header(VERSION_COEFF, cg.dims) + coeffs.astype("<i4").tobytes())


def read_coefficients(path) -> CoefficientGrid:
    """Read a version-2 coefficient file (coefficients.py:189-197); values
    outside the attainable range are a CorruptionError."""
    payload, dims = _read_payload(path, VERSION_COEFF, "<i4")
    lo, hi = COEFF_RANGE[len(dims)]
    if payload.size and (payload.min() < lo or payload.max() > hi):
        raise CorruptionError(f"{path}: coefficient outside [{lo}, {hi}] for a {len(dims)}D grid")
    return CoefficientGrid(payload.astype(np.int8).reshape(dims))


def write_curve(curve: EulerCurve, path) -> None:
    """``threshold,chi`` CSV; integers for exact curves, 9 significant digits
    otherwise (grid.py:300-307)."""
    taus, values = np.asarray(curve.taus, dtype=np.float64), np.asarray(curve.values)
    lines = ["threshold,chi"]
    if curve.is_integral:
        lines += [f"{t!r},{int(v)}" for t, v in zip(taus.tolist(), values.tolist())]
    else:
        lines += [f"{t!r},{v:.9g}" for t, v in zip(taus.tolist(), values.tolist())]
    Path(path).write_text("\n".join(lines) + "\n")


def read_curve(path) -> EulerCurve:
    """Read a curve CSV written by write_curve (grid.py:310-323)."""
    path = Path(path)
    lines = path.read_text().strip().splitlines()
    if not lines or lines[0].strip() != "threshold,chi":
        raise FormatError(f"{path}: first line must be 'threshold,chi'")
    taus, raw = [], []
    for line in lines[1:]:
        t, v = line.split(",")
        taus.append(float(t))
        raw.append(v)
    integral = all("." not in v and "e" not in v and "E" not in v for v in raw)
    values = (np.array([int(v) for v in raw], dtype=np.int64) if integral
              else np.array([float(v) for v in raw], dtype=np.float64))
    return EulerCurve(np.array(taus), values)


# ---------------------------------------------------------------------------
# streaming loader


def _readinto_exact(f, mv: memoryview, path) -> None:
    got = 0
    while got < len(mv):
        n = f.readinto(mv[got:])
        if not n:
            raise CorruptionError(f"{path}: payload ends early")
        got += n


def load_grid_device(path, device=None, planes: tuple[int, int] | None = None,
                     chunk_bytes: int = 64 << 20, check_finite: bool = True) -> torch.Tensor:
    """float32 tensor on `device` (default: the current CUDA device) holding
    the file's payload, or only planes [z0, z1) of axis 0.

    The payload streams through two pinned host buffers: while chunk k is
    copied host-to-device on a side stream, chunk k + 1 is read from the file.
    The caller's current stream is ordered after the copies.  Non-finite
    values raise ValueError, as ScalarGrid does (grid.py:63-64)."""
    h = read_header(path, VERSION_SCALAR, 4)
    dims = h.dims
    plane = h.count // dims[0]
    z0, z1 = (0, dims[0]) if planes is None else (int(planes[0]), int(planes[1]))
    if not (0 <= z0 <= z1 <= dims[0]):
        raise ValueError(f"plane range [{z0}, {z1}) outside [0, {dims[0]})")
    shape = (z1 - z0,) + tuple(dims[1:])
    n = (z1 - z0) * plane
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    out = torch.empty(shape, dtype=torch.float32, device=dev)
    flat = out.view(-1)
    with open(path, "rb", buffering=0) as f:
        f.seek(h.offset + 4 * z0 * plane)
        if dev.type != "cuda":
            _readinto_exact(f, memoryview(flat.numpy()).cast("B"), path)
        else:
            chunk = max(1, min(n, chunk_bytes // 4))
            bufs = [torch.empty(chunk, dtype=torch.float32, pin_memory=True) for _ in range(2 if n > chunk else 1)]
            done = [None] * len(bufs)
            side = torch.cuda.Stream(dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            pos, k = 0, 0
            while pos < n:
                m = min(chunk, n - pos)
                i = k % len(bufs)
                if done[i] is not None:
                    done[i].synchronize()        # the copy that last used this buffer
                _readinto_exact(f, memoryview(bufs[i].numpy()).cast("B")[:4 * m], path)
                with torch.cuda.stream(side):
                    flat[pos:pos + m].copy_(bufs[i][:m], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(side)
                done[i] = ev
                pos += m
                k += 1
            torch.cuda.current_stream(dev).wait_stream(side)
            for ev in done:
                if ev is not None:
                    ev.synchronize()             # pinned buffers are freed on return
    if check_finite and n:
        if dev.type == "cuda":
            from .hard import device_minmax

            _, _, bad = device_minmax(out)
        else:
            bad = int((~torch.isfinite(out)).sum())
        if bad:
            raise ValueError(f"{path}: grid values must be finite ({bad} non-finite)")
    return out


def load_slab_device(path, rank: int, world: int, device=None, **kw) -> tuple[torch.Tensor, tuple[int, int]]:
    """(padded, (z0, z1)) for rank `rank` of a `world`-way z-slab partition of
    a 3D grid file: padded[1:-1] = planes [z0, z1), padded[0] / padded[-1] =
    planes z0 - 1 / z1 read from the file (left uninitialised at the volume's
    ends, where distributed.slab_view drops them).  Feed it to
    distributed.slab_histogram(..., exchange=False)."""
    from .distributed import alloc_padded_slab, slab_bounds

    h = read_header(path, VERSION_SCALAR, 4)
    if len(h.dims) != 3:
        raise ValueError("z-slab loading needs a 3D grid file")
    if world > h.dims[0]:
        raise ValueError(f"cannot split {h.dims[0]} planes over {world} ranks (every rank needs a plane)")
    z0, z1 = slab_bounds(h.dims[0], world, rank)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    padded = alloc_padded_slab(z1 - z0, h.dims[1:], torch.float32, dev)
    lo, hi = max(z0 - 1, 0), min(z1 + 1, h.dims[0])
    src = load_grid_device(path, dev, (lo, hi), **kw)
    padded[1 - (z0 - lo):1 - (z0 - lo) + (hi - lo)].copy_(src)
    return padded, (z0, z1)


def save_grid_device(t: torch.Tensor, path) -> None:
    """Write a (device) float32 2D/3D tensor as a version-1 grid file."""
    if t.ndim not in (2, 3):
        raise ValueError(f"grid must be 2D or 3D, got ndim={t.ndim}")
    write_grid(t.detach().to(torch.float32), path)
