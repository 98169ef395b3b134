"""B200-native POET-X orthogonal-equivalence training layer.

Drop-in GPU implementation of the reference package's hot path
(/root/reference/pkg/src/poetx: cnp.py, blockdiag.py, permute.py,
layer.py, optim.py).  Host code is Python/PyTorch (device memory, streams,
torch.distributed); all arithmetic on the path runs in hand-written
sm_100a kernels in libpoetx_b200.so reached through a C ABI
(include/poetx_b200.h).  There is no CPU fallback.
"""

from .audit import singular_values, spectral_norm, spectrum_audit
from .blockdiag import (
    BlockDiagonalFactor,
    apply_to_features,
    apply_to_weight_cols,
    apply_to_weight_rows,
    assemble_dense,
    orthogonality_error,
    segmented_outer,
)
from .checkpoint import load_checkpoint, save_checkpoint
from .cnp import (
    CnpCache,
    SkewParams,
    cayley_exact,
    cnp_backward,
    cnp_backward_tc,
    cnp_forward_tc,
    cnp_forward,
    num_pairs,
    packed_grad_from_skew_grad,
    skew_from_packed,
)
from .errors import (
    CheckpointError,
    ConfigError,
    ConvergenceError,
    DataError,
    NumericsError,
    PoetxError,
    ShapeError,
    StateError,
)
from .layer import LayerCache, LayerGrads, MergeAudit, PoetLinearLayer, init_layer
from .optim import (
    AdamWState,
    ScheduleConfig,
    adamw_init,
    adamw_step,
    clip_threshold_at,
    fused_clip_adamw,
    global_clip,
    global_grad_norm,
    lr_at,
)
from .permute import (
    PermutationMap,
    dense_matrix,
    permute_cols,
    permute_features,
    permute_rows,
    premerge_weight,
    sample_permutation,
)
from .quant import QuantizedMatrix
from .rng import Rng

__version__ = "0.1.0"
