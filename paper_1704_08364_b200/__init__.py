"""B200-native BST filtered backprojection (arXiv:1704.08364), a drop-in for
the reference ``tomoblocks`` reconstruction API on sm_100a GPUs.

Modules mirror the reference layout: ``grids`` (slice containers),
``fourier_bp`` (BstPlan / FilterPlan / ramp_filter / bst_backproject / fbp /
fbp_volume), ``projector`` (backproject_ss), ``pipeline`` (StageSpec stages),
``phantom`` (synthetic inputs).  Compute runs in ``lib/libtb_bst.so``
(include/tb_bst.h); there is no CPU fallback.
"""

from .slices import (AngleAxis, DetectorAxis, ImageGrid, Sinogram, StageKind,  # noqa: F401
                     VolumeBlock, detector_coordinate, pixel_center)

__version__ = "0.1.0"


def __getattr__(name):
    # lazy: importing torch-backed modules only when the API is used
    if name in ("fourier_bp", "projector", "pipeline", "phantom", "preprocess", "slabs", "volio"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
