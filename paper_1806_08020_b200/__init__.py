"""B200-native polynomial-preconditioned thick-restart Arnoldi (PP-Arnoldi).

Python mirror of the reference's C++ entry points (arxiv/paper_1806_08020,
proj/include/ppa/*.hpp) over the C-ABI of libppa_b200.so (include/ppa_b200.h).
Every hot loop (pi(A)v, CGS2, V*Q) runs as hand-written sm_100a CUDA; there is
no CPU fallback: if the library is missing, importing the bindings raises.

Vectors passed to ``apply``/``apply_poly``/``build_gmres_poly`` are device
vectors: anything exposing ``data_ptr()`` (a torch CUDA tensor) or a raw int
device pointer.  ``apply_host`` is the end-to-end call with host numpy arrays.
"""
from __future__ import annotations

from ._capi import (  # noqa: F401
    CostRecord,
    CsrMatrix,
    LinearOperator,
    ArnoldiState,
    SolveConfig,
    PPAError,
    LogicError,
    lib,
    make_csr_operator,
    make_diagonal,
    make_poly_operator,
    make_poly_complement_operator,
    apply_poly,
    build_gmres_poly,
    leja_order,
    compute_pof,
    add_stability_roots,
    eval_poly,
    arnoldi_init,
    solve,
    solve_double,
    normal_vector,
    set_stream,
    synchronize,
    cgs2_step,
    ts_combine,
    spmv,
    spmm,
    check_ideal_order,
    damping_heuristic,
    make_block2,
    make_shifted,
    make_callback_operator,
    build_two_vector_poly,
    damped_start,
    read_matrix_market,
    STREAM_NORM,
    STREAM_POLY,
    STREAM_ARNOLDI,
    STREAM_POLY2,
    STREAM_MATRIX,
    SMALLEST_MAGNITUDE,
    LARGEST_MAGNITUDE,
    TARGET_ONE,
)
from .configs import CONFIGS, config_solve_config  # noqa: F401
