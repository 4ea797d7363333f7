"""CPU oracle for the ELSA FP32 attention path — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the reference package ``scanattn``
(/root/reference/pkg/src/scanattn) for the one hot path this repository
accelerates. It is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it. The CUDA path
(``paper_2604_23798_b200``) never imports this package and has no CPU
fallback.

Parity is pinned: ``tests/golden/*.npz`` hold outputs of the reference itself
(generated in the build container by ``tests/golden/make_golden.py``, which
imports /root/reference read-only), and ``tests/test_oracle.py`` checks every
function here against them bit-for-bit where the reference is deterministic
(generator, depth table, monoid KATs, FP64 naive attention, FP32 scan port).

Third-party algorithm dependency: the reference draws inputs with numpy's
``Philox`` bit generator and ``Generator.standard_normal`` (ziggurat),
``numpy>=1.24`` (pkg/pyproject.toml:10; 2.3.5 in this image). The restated
generator calls the same numpy primitives with the reference's keying and is
pinned by the golden Q/K/V fixtures.
"""

from .monoid import (  # noqa: F401
    identity_state,
    merge,
    merge_lanes,
    merge_tree,
)
from .problems import (  # noqa: F401
    SCENARIOS,
    depth_cap,
    generate,
    scan_depth,
)
from .attention import (  # noqa: F401
    U32,
    bound_threshold,
    naive_attention,
    naive_attention_rows_fp64,
    partial_state_fp64,
    row_err_conditioned,
    row_rel_err,
    sampled_rows_fp64,
    vectorized_probs,
)
from .scan_port import scan_forward_port  # noqa: F401
from .blocks import blockwise_states_fp64, inter_block_combine  # noqa: F401
