"""B200-native greedy binary-code construction (arXiv 1507.05398) -- Python binding.

A thin ctypes layer over ``libgc.so`` (C ABI: ``include/gc.h``).  Every function
here only marshals arguments; every step of the construction runs in the library's
sm_100a kernels.  PyTorch is used only for device memory and streams (the
``*_device`` / ``gc_generate_rank`` entry points take tensors).

If ``libgc.so`` is missing this module raises ImportError -- there is no CPU
fallback anywhere in the product path.
"""
from __future__ import annotations

from ._binding import (  # noqa: F401
    GC_FLAG_FORCE_SEQ_RESOLVE,
    GC_FLAG_KERNEL_TIMING,
    GC_FLAG_LAUNCHED_TILES,
    GC_FLAG_NO_EARLY_EXIT,
    GC_FLAG_NO_BLOCK_BOUND,
    GC_FLAG_NO_WEIGHT_BOUND,
    GC_FLAG_POPC_ONLY,
    GC_FLAG_SYNC_TILES,
    GC_FLAG_TILE_BARRIERS,
    GC_FLAG_NO_PREP,
    GC_FLAG_SIZE_ON_TRUE,
    GC_FLAG_NO_PARITY_BOUND,
    GC_FLAG_CROSS,
    GC_FLAG_NO_CATCHUP,
    GC_FLAG_CATCHUP,
    GC_FLAG_PIPELINED,
    GC_FLAG_STAGE_B,
    GC_FLAG_DEBUG_PHASES,
    GC_FLAG_NO_SUP_SMEM,
    GC_B_ORDERING,
    GC_GRADED_LEX,
    GC_GRADED_REVLEX,
    GC_GRAY,
    GC_LEX,
    ORDERINGS,
    GCError,
    LIB_PATH,
    exported_symbols,
    gc_abi_version,
    GcComm,
    gc_analyze,
    gc_analyze_device,
    gc_capacity_bound,
    gc_comm_attach_peers,
    gc_comm_create,
    gc_comm_destroy,
    gc_construct,
    gc_construct_device,
    gc_generate,
    gc_generate_device,
    gc_generate_ex,
    gc_generate_rank,
    gc_last_error,
    gc_nccl_id_bytes,
    gc_nccl_unique_id,
    gc_peer_handle_bytes,
    gc_peer_handles,
    gc_rank_to_vector,
    gc_ranks_to_vectors,
    gc_ranks_to_vectors_device,
    gc_strerror,
    gc_tile_partition,
    gc_vector_to_rank,
    ordering_id,
)

__all__ = [n for n in dir() if n.startswith("gc_") or n.startswith("GC_")] + [
    "GCError", "GcComm", "ORDERINGS", "ordering_id", "LIB_PATH", "exported_symbols"]
