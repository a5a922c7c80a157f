"""paper_2602_19090_b200 — B200-native forward-error-oriented eigenvector refinement (arXiv 2602.19090).

The product is the C-ABI library libozr.so (include/ozr.h) built from csrc/ for sm_100a; this package
is its thin Python binding (argument marshalling only). See DESIGN.md.
"""
from ._ozr import (OZR_COLWISE, OZR_ROWWISE, OZR_SPLIT_FIXED, OZR_SPLIT_X1, Comm, Context, OzrError, Params,
                   StepReport, colmajor, default_params, lib, ozr_comm_create_host_group, ozr_comm_create_nccl,
                   ozr_comm_nccl_id, ozr_gemm, ozr_gemm_plan, ozr_last_clusters, ozr_last_R, ozr_syev, ozr_syev_tridiag, ozr_syev_tridiag_eig, ozr_refine_step, ozr_refine_step_dist, ozr_refine_step_herm,
                   ozr_refine_to_tol, ozr_refine_to_tol_dist, ozr_split, ozr_version)

__all__ = ["Comm", "ozr_comm_create_host_group", "ozr_comm_create_nccl", "ozr_comm_nccl_id", "ozr_refine_step_dist",
           "ozr_refine_to_tol_dist", "Context", "OzrError", "Params", "StepReport", "colmajor", "default_params", "lib", "ozr_gemm",
           "ozr_gemm_plan", "ozr_last_clusters", "ozr_last_R", "ozr_syev", "ozr_syev_tridiag", "ozr_syev_tridiag_eig", "ozr_refine_step", "ozr_refine_step_herm", "ozr_refine_to_tol", "ozr_split", "ozr_version", "OZR_COLWISE",
           "OZR_ROWWISE", "OZR_SPLIT_FIXED", "OZR_SPLIT_X1"]
