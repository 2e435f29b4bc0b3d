"""B200-native Occupancy-Based Dual Contouring (ODC) mesh extraction.

Drop-in for the reference's extraction entry point
``occmesh.pipeline.contour(field, grid, options=None, counter=None)``
(/root/reference/pkg/src/occmesh/pipeline.py:154-240): same signature,
options, result type, stats and eval accounting, executed by hand-written
sm_100a kernels in libodc.so behind the C-ABI of include/odc.h.
"""

from .fields import (  # noqa: F401
    BoxField,
    CsgField,
    MeshWindingField,
    MlpField,
    OccupancyField,
    PlaneField,
    Scene,
    SmoothedOccupancy,
    SphereField,
    SurfaceCoincidenceError,
    TorusField,
    VoxelField,
    field_from_dict,
    load_scene,
    rotation_from_euler,
)
from .mesh import GridSpec, TriangleMesh  # noqa: F401
from .pipeline import (  # noqa: F401
    STATUS_NAMES,
    ConfigurationError,
    ContourOptions,
    ContourResult,
    EvalCounter,
    InternalContractError,
    LineBudget,
    SearchBudget,
    SharedField,
    contour,
    eval_labels,
    eval_raw,
)

__version__ = "0.1.0"
