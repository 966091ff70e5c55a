"""sigattn-b200: padding-aware bidirectional sigmoid attention (arxiv 2604.27124) on B200 / sm_100a.

Hot path: libsigattn.so (include/sigattn.h) -- hand-written tcgen05/TMEM/TMA kernels.
This package is the thin Python boundary (argument marshalling) plus the multi-GPU plumbing.
"""
from .attention import (sigattn_bwd, sigattn_fwd, sigattn_mask_to_seqlens, sigmoid_attention,  # noqa: F401
                        valid_flops, worklist_host, bwd_workspace_bytes, fwd_workspace_bytes, resolve_bias, sigattn_mask_to_index,
                        sigattn_permute_rows, copy_valid_rows)

__all__ = ["sigattn_fwd", "sigattn_bwd", "sigattn_mask_to_seqlens", "sigmoid_attention", "valid_flops",
           "worklist_host", "bwd_workspace_bytes", "fwd_workspace_bytes", "resolve_bias", "sigattn_mask_to_index", "sigattn_permute_rows",
           "copy_valid_rows"]
