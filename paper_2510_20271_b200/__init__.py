"""B200-native Euler Characteristic Curve engine (drop-in for ecckit's hot paths).

Same names and semantics as the reference package's hot-path API
(ecckit/__init__.py:11-117): exact curves (compute_ecc & co.) and the soft,
differentiable curve (soft_ecc / soft_ecc_backward), computed by sm_100a CUDA
kernels behind a C ABI (include/ecc_b200.h).  Torch-native extensions:
``ecc_discrete`` (batched exact curves on device tensors) and the
``SoftECC`` nn.Module.  Multi-GPU helpers live in ``.distributed``; grid files and
the streaming device loader in ``.io``.
"""

from .coefficients import COEFF_RANGE, CoefficientGrid, coefficients_device, compute_coefficients, vertex_order
from .grid import (
    CorruptionError,
    EulerCurve,
    FormatError,
    ScalarGrid,
    ThresholdSet,
    flatten_index,
    thresholds_from_range,
    unflatten_index,
    uniform_thresholds,
)
from .hard import (
    Chunked,
    FullSweep,
    HistogramBins,
    accumulate_histogram,
    bin_index,
    compute_ecc,
    device_minmax,
    ecc_discrete,
    ecc_discrete_host,
    release_host_buffers,
    histogram_device,
    merge_histograms,
    parse_strategy,
    scan_device,
)
from .io import (
    MAGIC,
    VERSION_COEFF,
    VERSION_SCALAR,
    load_grid_device,
    load_slab_device,
    read_coefficients,
    read_curve,
    read_grid,
    save_grid_device,
    write_coefficients,
    write_curve,
    write_grid,
)
from .soft import (
    SoftECC,
    SoftECCFunction,
    SoftEccParams,
    SoftGradients,
    effective_field,
    gradient_check,
    pixel_coordinates,
    reparametrize_direction,
    reparametrize_direction_jvp,
    soft_ecc,
    soft_ecc_backward,
    soft_step_host,
)

__version__ = "0.1.0"

__all__ = [
    "COEFF_RANGE", "CoefficientGrid", "Chunked", "CorruptionError", "EulerCurve", "FormatError", "FullSweep",
    "HistogramBins", "ScalarGrid", "SoftECC", "SoftECCFunction", "SoftEccParams", "SoftGradients", "ThresholdSet",
    "accumulate_histogram", "bin_index", "coefficients_device", "compute_coefficients", "compute_ecc",
    "device_minmax", "ecc_discrete", "ecc_discrete_host", "release_host_buffers", "effective_field", "flatten_index", "histogram_device", "merge_histograms",
    "parse_strategy", "pixel_coordinates", "reparametrize_direction", "reparametrize_direction_jvp", "scan_device",
    "soft_ecc", "soft_ecc_backward", "soft_step_host", "thresholds_from_range", "unflatten_index", "uniform_thresholds",
    "vertex_order", "gradient_check", "MAGIC", "VERSION_COEFF", "VERSION_SCALAR", "load_grid_device", "load_slab_device",
    "read_coefficients", "read_curve", "read_grid", "save_grid_device", "write_coefficients", "write_curve",
    "write_grid",
]
