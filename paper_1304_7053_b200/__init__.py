"""B200-native batched small-matrix GEMM (arXiv:1304.7053, Jhurani & Mullowney).

C^p <- alpha * op(A^p) op(B^p) + beta * C^p for thousands to millions of
independent triples with m, n, k <= 16, types s/d/c/z, ops N/T/C, strided
(second leading dimension) and pointer-array batches.  The compute path is the
C-ABI library libtxgemm.so (include/txgemm.h, CUDA for sm_100a); this package
is its thin binding (binding.py) plus the host-side work model (model.py).
"""
from . import model  # noqa: F401
from .binding import (TxError, build, gemm_batched, gemm_batched_ptr, last_path, prepare, lib, num_instances, set_tuning,  # noqa: F401,E501
                      pointer_array, set_max_ctas, status_string, tx_gemm_batched,
                      tx_gemm_batched_dev, tx_gemm_batched_hostio, tx_gemm_batched_ptr,
                      tx_gemm_batched_ptr_dev, version)
from .binding import (tx_gemm_batched_s, tx_gemm_batched_d, tx_gemm_batched_c,  # noqa: F401
                      tx_gemm_batched_z, tx_gemm_batched_ptr_s, tx_gemm_batched_ptr_d,
                      tx_gemm_batched_ptr_c, tx_gemm_batched_ptr_z, tx_gemm_batched_hostio_s,
                      tx_gemm_batched_hostio_d, tx_gemm_batched_hostio_c,
                      tx_gemm_batched_hostio_z)

__all__ = ["gemm_batched", "gemm_batched_ptr", "prepare", "model", "lib", "build"]
