"""B200-native edge-server view synthesis (FVV Live, arXiv 2007.00558).

Host-side mirror of the reference package's synthesis API over the C ABI of
``libfvvb200.so`` (``include/fvv_b200.h``). Submodules:

* ``types``, ``geometry``, ``selection`` — rig API (host, no kernels);
* ``synthesis`` — drop-in for ``fvv.synthesis`` (GPU);
* ``depthproc`` / ``depthcodec`` — edge-server depth preprocessing (GPU);
* ``engine`` — resident-slot session renderer and ``synthesize()``;
* ``scenes`` — seeded synthetic MVD workloads (test/bench inputs);
* ``pytest_shim`` — routes ``fvv.synthesis`` to this package.

Compute modules import torch lazily through ``_dev``; the rig API works
without a GPU.
"""

__version__ = "0.1.0"

from .geometry import (build_camera_arc, camera_distance, load_rig, look_at_pose,  # noqa: F401
                       save_rig)
from .selection import select_cameras, select_references  # noqa: F401
from .types import (CameraCalibration, CameraIntrinsics, CameraPose, ColorFrame,  # noqa: F401
                    DepthFrame, DepthRange, MvdFrame, Validity)


def __getattr__(name):
    if name in ("EdgeRenderer", "synthesize"):
        from . import engine
        return getattr(engine, name)
    if name == "SynthesisConfig":
        from .synthesis import SynthesisConfig
        return SynthesisConfig
    raise AttributeError(name)
