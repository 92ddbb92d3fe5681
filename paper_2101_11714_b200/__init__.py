"""B200-native TT-EmbeddingBag (TT-Rec, arXiv:2101.11714): a drop-in for the
reference C++ operator's hot path, implemented as sm_100a CUDA kernels behind
a C ABI (include/ttgpu.h, lib/libttgpu.so)."""
from .ttrec import (  # noqa: F401
    CoreGradients,
    EmbeddingStats,
    ForwardContext,
    ForwardResult,
    IndexBatch,
    InvalidArgument,
    OutOfRange,
    Pooling,
    RuntimeFailure,
    ShapePlan,
    TtTable,
    backward_bags,
    decompose_index,
    forward_bags,
    generate_zipfian_batch,
    kDefaultMicroBatch,
    lookup_row,
    plan_shapes,
    recompose_index,
    sgd_step,
    uniform_indices,
    derived_uniform_indices,
)
from . import lfu_cache  # noqa: F401,E402
from .lfu_cache import (  # noqa: F401,E402
    CachePartition,
    CacheState,
    EmbeddingLayer,
    FreqTable,
    LfuCache,
    hot_set_drift,
)
from . import sharding  # noqa: F401,E402
from . import checkpoint  # noqa: F401,E402
from . import streams  # noqa: F401,E402
from . import collection  # noqa: F401,E402
from . import dense  # noqa: F401,E402
