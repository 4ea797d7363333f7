"""ELSA on B200: exact FP32 softmax attention as an associative (m, S, W)
state reduction (arXiv 2604.23798), computed by hand-written sm_100a CUDA
kernels behind a C-ABI (include/elsa.h, libelsa.so).

Entry points:
  * scaled_dot_product_attention(q, k, v) — drop-in for
    torch.nn.functional.scaled_dot_product_attention on (B, H, n, d) FP32
    CUDA tensors;
  * attention_from_host(q, k, v) — the same on HOST arrays, with the
    host<->device copies pipelined under the kernels (elsa_fwd_f32_host);
  * partial_states / merge_states — per-key-range (m, S, W) summaries and
    their fixed (+)-tree merge (Proposition 1), the building blocks of the
    KV-sharded multi-GPU path in ``paper_2604_23798_b200.dist``;
  * scanattn_compat.scan_forward(problem, cfg) — the reference engine's
    signature (engine.py:385-427) on the GPU.
"""

from .attention import (  # noqa: F401
    attention_from_host,
    blockwise_states,
    inter_block_combine,
    check_device_error,
    describe_plan,
    ffma_peak_tflops,
    last_launch_count,
    merge_peer_states,
    merge_states,
    partial_states,
    resolve_kv_splits,
    scaled_dot_product_attention,
)
from .errors import (  # noqa: F401
    ElsaCudaError,
    ElsaLibraryError,
    NumericalError,
    ShapeError,
    WorkspaceError,
)

__version__ = "0.1.0"
