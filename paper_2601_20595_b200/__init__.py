"""B200-native AutoOverlap hot path: fused AllGather->GEMM and GEMM->ReduceScatter
kernels for sm_100a, scheduled at communication-chunk granularity (arXiv 2601.20595).

Also the NEXT rows: GEMM-AllReduce, the MoE All-to-All dispatch + expert GEMM, and
sequence-parallel (ring-ordered) and head-parallel (all-to-all) attention.
The compute path is the C-ABI library libautooverlap.so (include/autooverlap.h); this
package is its thin Python binding.  There is no CPU fallback.
"""
from .api import (AOError, Context, Plan, a2a_gemm, a2a_gemm_group, ag_gemm, ag_gemm_group, debug_set, device_query, dist_world, transfer_bench,  # noqa: F401
                  gemm, gemm_ar, gemm_ar_group, gemm_batched, gemm_rs, gemm_rs_group, group_schedule_json, hp_attn, hp_attn_group, loopback_world, plan_json, sp_attn, sp_attn_group, validate,
                  workspace_bytes)

__all__ = ["AOError", "Context", "Plan", "a2a_gemm", "a2a_gemm_group", "ag_gemm", "ag_gemm_group", "gemm", "gemm_ar", "gemm_ar_group", "gemm_batched", "gemm_rs", "gemm_rs_group", "sp_attn", "sp_attn_group", "hp_attn", "hp_attn_group",
           "loopback_world", "dist_world", "plan_json", "group_schedule_json", "validate", "workspace_bytes", "debug_set", "device_query", "transfer_bench"]
