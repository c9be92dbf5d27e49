"""B200-native (sm_100a, FP64) tiled Gaussian-process hot path.

Drop-in for the reference ``taskgp`` model API (pkg/src/taskgp/__init__.py),
computing on hand-written CUDA kernels through the C ABI in
``include/gpb200.h``::

    import paper_2505_00136_b200 as gpb

    gpb.start_runtime(gpb.RuntimeConfig())
    model = gpb.GPModel(train, gpb.KernelParams(), tiles_per_dim=4)
    result = model.predict_variance(test)
    gpb.stop_runtime()
"""

from . import bench, errors
from .covariance import KernelParams
from .data import (
    Dataset,
    LagSpec,
    lag_embed,
    lag_features,
    load_csv,
    make_msd_dataset,
    make_msd_dataset_device,
    msd_series,
    save_csv,
)
from .model import GP, AdamConfig, GPModel, PredictionResult
from .runtime import (
    Runtime,
    RuntimeConfig,
    current_runtime,
    run_as_root,
    start_runtime,
    stop_runtime,
)
from .tiles import B200TileKernels

__version__ = "0.1.0"

__all__ = [
    "AdamConfig",
    "LagSpec",
    "bench",
    "lag_embed",
    "load_csv",
    "save_csv",
    "B200TileKernels",
    "Dataset",
    "GP",
    "GPModel",
    "KernelParams",
    "PredictionResult",
    "Runtime",
    "RuntimeConfig",
    "current_runtime",
    "errors",
    "lag_features",
    "make_msd_dataset",
    "make_msd_dataset_device",
    "msd_series",
    "run_as_root",
    "start_runtime",
    "stop_runtime",
    "__version__",
]
