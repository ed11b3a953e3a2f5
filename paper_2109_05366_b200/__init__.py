"""B200-native GPUfs-style sequential-read layer (readahead prefetcher + per-TB LRA).

Drop-in for the reference package ``gpuiosim``'s sequential gread path: the same
``ExperimentConfig`` keys, ``Simulation(cfg, seed).run() -> MetricsReport`` and
``SimError``, executed on real hardware (HBM page cache, pinned RPC ring, host
I/O daemon) by libgfs.so.  See DESIGN.md.
"""

import os as _os

# DMA transfers run the host daemon's copies on their own streams while the persistent
# gread kernel occupies another.  With the driver's default of 8 hardware work queues, a
# daemon stream can alias the kernel's queue and its copy (and the doorbell behind it)
# would wait for the kernel that waits for it.  Ask for enough queues before CUDA starts.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from .config import ExperimentConfig, load_config  # noqa: E402
from .errors import GfsError, SimError
from .rng import SeededRng

__version__ = "0.1.0"


def __getattr__(name):  # lazy: keep `import` cheap and torch-free until used
    if name in ("GpuFS", "Simulation", "ensure_synthetic", "O_RDONLY", "O_RDWR"):
        from . import runtime
        return getattr(runtime, name)
    raise AttributeError(name)


__all__ = ["ExperimentConfig", "load_config", "GfsError", "SimError", "SeededRng",
           "GpuFS", "Simulation", "ensure_synthetic", "__version__"]
