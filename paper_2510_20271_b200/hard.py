"""Exact Euler characteristic curves -- the API of ecckit/hard.py on the GPU.

``compute_ecc`` / ``accumulate_histogram`` keep the reference's signatures
(hard.py:184-226).  The reference's two strategies (FullSweep, Chunked) and
its worker count are accepted for compatibility; the device always runs one
fused sweep (ecc_histogram) whose integer result equals both strategies'
(strategy equivalence) at every worker count.

``ecc_discrete`` is the torch-native batched entry point: a CUDA tensor of
shape [N?, (D,) H, W] in, int64 curves [N?, B] out, no host round trip.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .grid import EulerCurve, ScalarGrid, ThresholdSet


@dataclass(frozen=True)
class FullSweep:
    """Single pass over the grid (hard.py:41-46)."""

    def __str__(self):
        return "fullsweep"


@dataclass(frozen=True)
class Chunked:
    """Sequential fixed-size chunks (hard.py:49-60).  Accepted for API
    compatibility; results are identical to FullSweep by construction."""

    chunk_len: int

    def __post_init__(self):
        if self.chunk_len < 1:
            raise ValueError(f"chunk_len must be >= 1, got {self.chunk_len}")

    def __str__(self):
        return f"chunked:{self.chunk_len}"


Strategy = FullSweep | Chunked


def parse_strategy(text: str) -> Strategy:
    """Parse ``fullsweep`` or ``chunked:<k>`` (hard.py:66-72)."""
    if text == "fullsweep":
        return FullSweep()
    if text.startswith("chunked:"):
        return Chunked(int(text.split(":", 1)[1]))
    raise ValueError(f"unknown strategy {text!r}; expected 'fullsweep' or 'chunked:<k>'")


@dataclass(frozen=True)
class HistogramBins:
    """Integer coefficient totals per threshold bin (hard.py:75-86)."""

    taus: np.ndarray
    bins: np.ndarray
    overflow: int


def bin_index(x: float, taus: ThresholdSet) -> int | None:
    """Smallest j with x <= taus[j], or None beyond the last (hard.py:89-96)."""
    j = int(np.searchsorted(taus.taus, x, side="left"))
    return j if j < len(taus) else None


def merge_histograms(parts) -> HistogramBins:
    """Element-wise int64 sum over identical threshold sets (hard.py:99-118)."""
    parts = list(parts)
    if not parts:
        raise ValueError("cannot merge zero histograms")
    first = parts[0]
    for p in parts[1:]:
        if p.bins.shape != first.bins.shape:
            raise ValueError(f"histogram bin counts differ: {p.bins.size} vs {first.bins.size}")
        if not np.array_equal(p.taus, first.taus):
            raise ValueError("histograms were accumulated over different thresholds")
    bins = np.sum([p.bins for p in parts], axis=0, dtype=np.int64)
    overflow = int(sum(p.overflow for p in parts))
    return HistogramBins(first.taus, bins, overflow)


# ---------------------------------------------------------------------------
# device primitives
# ---------------------------------------------------------------------------

def device_minmax(t: torch.Tensor) -> tuple[float, float, int]:
    """(min, max, #non-finite) of a CUDA tensor via ecc_minmax (one pass)."""
    L = _lib.lib()
    t = t.contiguous()
    out = torch.empty(3, dtype=torch.int64, device=t.device)
    _lib.check(L.ecc_minmax(_lib.ptr(t), _lib.dtype_code(t), t.numel(), _lib.ptr(out), _lib.stream_ptr(t)))
    k = out.cpu().numpy().view(np.uint64)
    return float(L.ecc_key_to_double(int(k[0]))), float(L.ecc_key_to_double(int(k[1]))), int(k[2])


def _split_batch(x: torch.Tensor, ndim: int | None):
    """(batch, grid dims) of a [N?, (D,) H, W] tensor."""
    if ndim is None:
        ndim = x.ndim if x.ndim in (2, 3) else None
        if ndim is None:
            raise ValueError(f"pass ndim for a {x.ndim}-D tensor (batched grids)")
    if ndim not in (2, 3):
        raise ValueError(f"grid must be 2D or 3D, got ndim={ndim}")
    if x.ndim == ndim:
        return 1, tuple(x.shape), False
    if x.ndim == ndim + 1:
        return int(x.shape[0]), tuple(x.shape[1:]), True
    raise ValueError(f"expected a {ndim}-D grid or a batch of them, got shape {tuple(x.shape)}")


def _binning_bytes(b) -> torch.Tensor:
    return torch.frombuffer(bytearray(bytes(b)), dtype=torch.uint8)


def _binning_from(t: torch.Tensor):
    return _lib.Binning.from_buffer_copy(t.numpy().tobytes())


# The fused sweep and the scan as torch.library custom ops (fake
# implementations give torch.compile the output shapes, no graph break).  The
# threshold table is built on the host (ThresholdSet.device_table) and passed
# in: a device table tensor plus the ecc_binning struct as a CPU byte tensor.
@torch.library.custom_op("ecc_b200::histogram", mutates_args=())
def _histogram_op(x: torch.Tensor, table: torch.Tensor, binning: torch.Tensor, ndim: int, nbins: int,
                  check_finite: bool) -> tuple[torch.Tensor, torch.Tensor]:
    """(int64 [N, B+1] histograms, int32 [1] non-finite flag) of x [N?, (D,) H, W]."""
    batch, dims, _ = _split_batch(x, ndim)
    hist = torch.empty((batch, nbins + 1), dtype=torch.int64, device=x.device)
    flag = torch.zeros(1, dtype=torch.int32, device=x.device)
    d = _lib.dims_arg(dims)
    b = _binning_from(binning)
    L = _lib.lib()
    if check_finite:
        _lib.check(L.ecc_histogram_checked(_lib.ptr(x), _lib.dtype_code(x), len(dims), _lib.ptr(d), batch, 0,
                                           dims[0] if len(dims) == 3 else 1, _lib.ptr(table), _lib.ctypes.byref(b),
                                           _lib.ptr(hist), _lib.ptr(flag), _lib.stream_ptr(x)))
    else:
        _lib.check(L.ecc_histogram(_lib.ptr(x), _lib.dtype_code(x), len(dims), _lib.ptr(d), batch, _lib.ptr(table),
                                   _lib.ctypes.byref(b), _lib.ptr(hist), _lib.stream_ptr(x)))
    return hist, flag


@_histogram_op.register_fake
def _(x, table, binning, ndim, nbins, check_finite):
    batch, _, _ = _split_batch(x, ndim)
    return x.new_empty((batch, nbins + 1), dtype=torch.int64), x.new_empty((1,), dtype=torch.int32)


@torch.library.custom_op("ecc_b200::scan", mutates_args=())
def _scan_op(hist: torch.Tensor, nbins: int) -> torch.Tensor:
    """Inclusive prefix over the first nbins columns -> int64 [N, B] curves."""
    batch = hist.shape[0]
    curve = torch.empty((batch, nbins), dtype=torch.int64, device=hist.device)
    _lib.check(_lib.lib().ecc_scan(_lib.ptr(hist), batch, nbins, _lib.ptr(curve), _lib.stream_ptr(hist)))
    return curve


@_scan_op.register_fake
def _(hist, nbins):
    return hist.new_empty((hist.shape[0], nbins), dtype=torch.int64)


def _hist(x: torch.Tensor, taus: ThresholdSet, ndim: int | None, check_finite: bool):
    if not x.is_cuda:
        raise ValueError("histogram_device takes a CUDA tensor")
    x = x.contiguous()
    _split_batch(x, ndim)   # validates the shape
    table, binning = taus.device_table(_lib.dtype_code(x), x.device)
    nd = ndim if ndim is not None else x.ndim
    return torch.ops.ecc_b200.histogram(x, table, _binning_bytes(binning), nd, len(taus), check_finite)


def _raise_nonfinite(flag: torch.Tensor) -> None:
    if int(flag.item()):
        raise ValueError("grid values must be finite (the device found NaN or Inf)")


def histogram_device(x: torch.Tensor, taus: ThresholdSet, ndim: int | None = None,
                     check_finite: bool = False) -> torch.Tensor:
    """int64 [N, B+1] coefficient histograms (last column = overflow) of CUDA
    grids x [N?, (D,) H, W] (uint8 / float32 / float64).  check_finite:
    raise ValueError for NaN / Inf values like ScalarGrid (grid.py:63-64);
    the float32 kernels test while they sweep, the raise reads a flag back."""
    hist, flag = _hist(x, taus, ndim, check_finite)
    if check_finite:
        _raise_nonfinite(flag)
    return hist


def scan_device(hist: torch.Tensor, nbins: int) -> torch.Tensor:
    """Inclusive prefix over the first nbins columns -> int64 [N, B] curves."""
    return torch.ops.ecc_b200.scan(hist, nbins)


def ecc_discrete(x: torch.Tensor, taus, ndim: int | None = None, return_hist: bool = False,
                 check_finite: bool = True):
    """Torch-native batched exact ECC.

    x: CUDA tensor [N?, (D,) H, W] of uint8 / float32 / float64 (float32
    values are compared exactly as the reference's float64 would be).
    taus: ThresholdSet or 1-D array of strictly increasing thresholds.
    Returns int64 curves [N?, B] on the device (and the [N?, B+1] histogram).
    NaN / Inf values raise ValueError like ScalarGrid (grid.py:63-64); the
    check runs inside the fused sweep, and reading its flag is one small
    device -> host copy (check_finite=False skips it: fully asynchronous).
    """
    ts = taus if isinstance(taus, ThresholdSet) else ThresholdSet(taus)
    _, _, batched = _split_batch(x, ndim)
    hist, flag = _hist(x, ts, ndim, check_finite)
    curve = scan_device(hist, len(ts))
    if check_finite:
        _raise_nonfinite(flag)
    if not batched:
        curve, hist = curve[0], hist[0]
    return (curve, hist) if return_hist else curve


class _StreamState:
    """Device buffers of ecc_discrete_host, one cached configuration per
    (calling thread, device stream): concurrent calls from different threads
    or on different streams never share a buffer, and calls on one stream are
    ordered by the stream (plus the event recorded after each call's last
    kernel, waited on before the next call's first copy)."""

    _local = threading.local()

    @classmethod
    def table(cls) -> dict:
        t = getattr(cls._local, "cache", None)
        if t is None:
            t = cls._local.cache = {}
        return t

    @classmethod
    def get(cls, stream, key):
        st = cls.table().get(stream.cuda_stream)
        return st if st is not None and st.get("key") == key else None

    @classmethod
    def put(cls, stream, st):
        cls.table()[stream.cuda_stream] = st   # one configuration per stream: the previous one is freed


def release_host_buffers() -> None:
    """Free the device buffers ecc_discrete_host keeps for this thread's streams."""
    _StreamState.table().clear()


RESIDENT_MAX_BYTES = 8 << 30   # ecc_discrete_host(resident=None): volumes up to this size stay in HBM


def ecc_discrete_host(x_host: torch.Tensor, taus, chunk_planes: int = 64, device=None, return_hist: bool = False,
                      resident=None):
    """Exact ECC of a 3D volume held in HOST memory, streamed to the GPU.

    The volume (float32 / uint8 / float64, [D, H, W], row-major) is cut into
    z-chunks of ``chunk_planes`` planes whose host-to-device copies run on a
    copy stream while the fused kernel (ecc_histogram_range) deposits the
    planes already on the device, so the end-to-end time is the larger of
    the PCIe transfer and the compute instead of their sum.  Two layouts:

    * resident (default for volumes up to RESIDENT_MAX_BYTES): the chunks
      land in one device copy of the volume, every plane crosses PCIe once,
      and after chunk k arrives the kernel deposits every plane whose z + 1
      neighbour is on the device; only the last chunk's deposit follows the
      last copy, so small chunks leave a short tail.
    * ring (``resident=False``, or larger volumes): two (chunk + 2)-plane
      device buffers, each chunk copied with its one-plane halos, so the
      volume need not fit in device memory.

    Pass pinned memory (``tensor.pin_memory()``) for asynchronous copies.
    The result equals ecc_discrete(x_host.cuda(), taus) bit for bit
    (histograms are exactly additive over planes, hard.py:99-118; the
    tie-break is translation invariant, coefficients.py:141-152).
    """
    if isinstance(x_host, np.ndarray):
        x_host = torch.from_numpy(np.ascontiguousarray(x_host))
    if x_host.is_cuda or x_host.ndim != 3:
        raise ValueError("ecc_discrete_host takes a 3-D host tensor")
    if chunk_planes < 1:
        raise ValueError(f"chunk_planes must be >= 1, got {chunk_planes}")
    x_host = x_host.contiguous()
    ts = taus if isinstance(taus, ThresholdSet) else ThresholdSet(taus)
    dev = torch.device(device) if device is not None else _lib.device()
    D, H, W = (int(d) for d in x_host.shape)
    code = _lib.dtype_code(x_host)
    nb = len(ts)
    table, binning = ts.device_table(code, dev)
    cp = min(chunk_planes, D)
    auto = resident is None
    if auto:
        resident = x_host.numel() * x_host.element_size() <= RESIDENT_MAX_BYTES
    if resident:
        try:
            return _ecc_discrete_host_resident(x_host, ts, cp, dev, code, table, binning, return_hist)
        except torch.cuda.OutOfMemoryError:
            if not auto:
                raise
            release_host_buffers()   # no room for the whole volume: stream through the ring
            torch.cuda.empty_cache()
    main = torch.cuda.current_stream(dev)
    key = (x_host.dtype, cp, H, W, nb, str(dev))
    st = _StreamState.get(main, key)
    if st is None:
        st = {"key": key, "bufs": [torch.empty((cp + 2, H, W), dtype=x_host.dtype, device=dev) for _ in range(2)],
              "part": [torch.empty(nb + 1, dtype=torch.int64, device=dev) for _ in range(2)],
              "copy": torch.cuda.Stream(dev), "done": None}
        _StreamState.put(main, st)
    cs = st["copy"]
    total = torch.zeros(nb + 1, dtype=torch.int64, device=dev)
    freed = [None, None]
    cs.wait_stream(main)
    if st["done"] is not None:
        cs.wait_event(st["done"])   # the previous call's kernels are done with the buffers
    for c, z0 in enumerate(range(0, D, cp)):
        z1 = min(z0 + cp, D)
        lo, hi = max(z0 - 1, 0), min(z1 + 1, D)
        buf, part = st["bufs"][c % 2], st["part"][c % 2]
        with torch.cuda.stream(cs):
            if freed[c % 2] is not None:
                cs.wait_event(freed[c % 2])       # the kernel that last read this buffer is done
            buf[:hi - lo].copy_(x_host[lo:hi], non_blocking=True)
            copied = torch.cuda.Event()
            copied.record(cs)
        main.wait_event(copied)
        view = buf[:hi - lo]
        d = _lib.dims_arg(view.shape)
        _lib.check(_lib.lib().ecc_histogram_range(_lib.ptr(view), code, 3, _lib.ptr(d), 1, z0 - lo, z1 - lo,
                                                  _lib.ptr(table), _lib.ctypes.byref(binning), _lib.ptr(part),
                                                  _lib.ctypes.c_void_p(main.cuda_stream)))
        total += part
        ev = torch.cuda.Event()
        ev.record(main)
        freed[c % 2] = ev
    curve = scan_device(total.reshape(1, -1), nb)[0]
    st["done"] = freed[(D - 1) // cp % 2]
    return (curve, total) if return_hist else curve


def _ecc_discrete_host_resident(x_host, ts, cp, dev, code, table, binning, return_hist):
    D, H, W = (int(d) for d in x_host.shape)
    nb = len(ts)
    nchunks = (D + cp - 1) // cp
    key = ("resident", x_host.dtype, D, H, W, nb, nchunks, str(dev))
    main = torch.cuda.current_stream(dev)
    st = _StreamState.get(main, key)
    if st is None:
        st = {"key": key, "vol": torch.empty((D, H, W), dtype=x_host.dtype, device=dev),
              "parts": torch.empty((nchunks, nb + 1), dtype=torch.int64, device=dev),
              "copy": torch.cuda.Stream(dev), "done": None}
        _StreamState.put(main, st)
    vol, parts, cs = st["vol"], st["parts"], st["copy"]
    d = _lib.dims_arg(vol.shape)
    cs.wait_stream(main)
    if st["done"] is not None:
        cs.wait_event(st["done"])   # the previous call's kernels are done with vol and parts
    a = 0                  # planes [0, a) deposited
    for k in range(nchunks):
        z0, z1 = k * cp, min((k + 1) * cp, D)
        with torch.cuda.stream(cs):
            vol[z0:z1].copy_(x_host[z0:z1], non_blocking=True)
            copied = torch.cuda.Event()
            copied.record(cs)
        main.wait_event(copied)
        b = D if z1 == D else z1 - 1   # plane p is deposited once plane p + 1 is on the device
        if b > a:
            _lib.check(_lib.lib().ecc_histogram_range(_lib.ptr(vol), code, 3, _lib.ptr(d), 1, a, b,
                                                      _lib.ptr(table), _lib.ctypes.byref(binning),
                                                      _lib.ptr(parts[k]), _lib.ctypes.c_void_p(main.cuda_stream)))
        else:
            parts[k].zero_()
        a = max(a, b)
    total = parts.sum(0)
    done = torch.cuda.Event()
    done.record(main)
    st["done"] = done
    curve = scan_device(total.reshape(1, -1), nb)[0]
    return (curve, total) if return_hist else curve


def _check_strategy(strategy, workers):
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    if not isinstance(strategy, (FullSweep, Chunked)):
        raise TypeError(f"unknown strategy {strategy!r}")


def accumulate_histogram(
    grid: ScalarGrid,
    taus: ThresholdSet,
    strategy: Strategy = FullSweep(),
    workers: int = 1,
) -> HistogramBins:
    """Coefficient histogram of a grid (hard.py:184-212), on the GPU."""
    _check_strategy(strategy, workers)
    h = histogram_device(grid.device_tensor(), taus)[0].cpu().numpy()
    return HistogramBins(taus.taus, h[:-1].copy(), int(h[-1]))


def compute_ecc(
    grid: ScalarGrid,
    taus: ThresholdSet,
    strategy: Strategy = FullSweep(),
    workers: int = 1,
) -> EulerCurve:
    """Exact Euler characteristic curve at every threshold (hard.py:215-226)."""
    _check_strategy(strategy, workers)
    curve = ecc_discrete(grid.device_tensor(), taus)
    return EulerCurve(taus.taus, curve.cpu().numpy())
