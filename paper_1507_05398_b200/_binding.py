"""ctypes marshalling for libgc.so (include/gc.h).  Names match the C ABI."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgc.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "gc.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
        "there is no CPU fallback for the greedy construction")

GC_LEX, GC_GRAY, GC_GRADED_LEX, GC_GRADED_REVLEX = 0, 1, 2, 3
ORDERINGS = {"lex": GC_LEX, "gray": GC_GRAY, "glex": GC_GRADED_LEX, "grlex": GC_GRADED_REVLEX,
             "graded-lex": GC_GRADED_LEX, "graded-revlex": GC_GRADED_REVLEX}
GC_FLAG_NO_EARLY_EXIT = 0x1
GC_FLAG_SYNC_TILES = 0x2
GC_FLAG_FORCE_SEQ_RESOLVE = 0x4
GC_FLAG_KERNEL_TIMING = 0x8
GC_FLAG_LAUNCHED_TILES = 0x10
GC_FLAG_POPC_ONLY = 0x20
GC_FLAG_NO_WEIGHT_BOUND = 0x40
GC_FLAG_NO_BLOCK_BOUND = 0x80
GC_FLAG_TILE_BARRIERS = 0x100
GC_FLAG_NO_PREP = 0x800
GC_FLAG_SIZE_ON_TRUE = 0x1000
GC_FLAG_NO_PARITY_BOUND = 0x2000
GC_FLAG_CROSS = 0x4000
GC_FLAG_NO_CATCHUP = 0x8000
GC_FLAG_CATCHUP = 0x10000
GC_FLAG_PIPELINED = 0x20000
GC_FLAG_STAGE_B = 0x40000
GC_FLAG_DEBUG_PHASES = 0x200
GC_FLAG_NO_SUP_SMEM = 0x400

_STATUS = {0: "GC_OK", 1: "GC_EINVAL", 2: "GC_ERANGE", 3: "GC_ENOSPC", 4: "GC_EUNSUPPORTED",
           5: "GC_ECUDA", 6: "GC_ENOMEM", 7: "GC_ENCCL", 8: "GC_EINTERNAL"}


class gc_options(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("tile_min", ctypes.c_uint32),
                ("tile_max", ctypes.c_uint32), ("window0", ctypes.c_uint32),
                ("emulate_ranks", ctypes.c_uint32), ("flags", ctypes.c_uint32),
                ("window_growth", ctypes.c_uint32), ("pipeline_depth", ctypes.c_uint32),
                ("target_accepted", ctypes.c_uint32), ("items_per_warp", ctypes.c_uint32),
                ("sub_max", ctypes.c_uint32), ("geo_head", ctypes.c_uint32), ("split_bits", ctypes.c_uint32),
                ("partial_s", ctypes.c_uint32), ("grid_ctas", ctypes.c_uint32), ("plan_warps", ctypes.c_uint32),
                ("prep_lead", ctypes.c_uint32), ("prep_ctas", ctypes.c_uint32), ("burst_chunk", ctypes.c_uint32)]


GC_B_ORDERING = 4


class gc_problem(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("n", ctypes.c_uint32), ("d", ctypes.c_uint32),
                ("ordering", ctypes.c_int32), ("basis", ctypes.POINTER(ctypes.c_uint64)),
                ("constant_weight", ctypes.c_int32), ("self_orthogonal", ctypes.c_uint32)]


class gc_stats(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("n_ranks", ctypes.c_uint32),
                ("device_ms", ctypes.c_double), ("wall_ms", ctypes.c_double),
                ("M", ctypes.c_uint64), ("tiles", ctypes.c_uint64), ("phases", ctypes.c_uint64),
                ("checks_exec", ctypes.c_uint64), ("survivors", ctypes.c_uint64),
                ("conflicts", ctypes.c_uint64), ("resolve_checks", ctypes.c_uint64),
                ("w_def", ctypes.c_double), ("launches", ctypes.c_uint64),
                ("screen_launches", ctypes.c_uint64), ("screen_ms", ctypes.c_double),
                ("bound_tests", ctypes.c_uint64), ("resolve_wait_ms", ctypes.c_double),
                ("resolve_busy_ms", ctypes.c_double), ("pipeline_depth", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32), ("prep_used", ctypes.c_uint64)]

    def to_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_ if name != "struct_size"}


class gc_analysis(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("min_distance", ctypes.c_uint32), ("M", ctypes.c_uint64),
                ("weight_hist", ctypes.c_uint64 * 33), ("gf2_rank", ctypes.c_uint32),
                ("is_linear", ctypes.c_uint32), ("self_orthogonal", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32), ("pairs_checked", ctypes.c_uint64)]

    def to_dict(self) -> dict:
        return {"M": self.M, "min_distance": self.min_distance, "gf2_rank": self.gf2_rank,
                "is_linear": bool(self.is_linear), "self_orthogonal": {0: False, 1: True}.get(self.self_orthogonal),
                "weights": {w: int(self.weight_hist[w]) for w in range(33) if self.weight_hist[w]},
                "pairs_checked": self.pairs_checked}


GC_ANALYZE_PAIRWISE = 0x1
GC_ANALYZE_ORTHOGONALITY = 0x2

_u64p = ctypes.POINTER(ctypes.c_uint64)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_lib = ctypes.CDLL(LIB_PATH)


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype, f.argtypes = res, args
    return f


_sig("gc_generate", ctypes.c_int, [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int, _u64p, _u64p])
_sig("gc_generate_ex", ctypes.c_int, [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int,
                                      ctypes.POINTER(gc_options), _u64p, _u64p, ctypes.POINTER(gc_stats)])
_sig("gc_generate_device", ctypes.c_int, [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int,
                                          ctypes.POINTER(gc_options), ctypes.c_void_p, ctypes.c_uint64,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(gc_stats)])
_sig("gc_capacity_bound", ctypes.c_uint64, [ctypes.c_uint32, ctypes.c_uint32])
_sig("gc_construct", ctypes.c_int, [ctypes.POINTER(gc_problem), ctypes.POINTER(gc_options), _u64p, _u64p,
                                    ctypes.POINTER(gc_stats)])
_sig("gc_construct_device", ctypes.c_int, [ctypes.POINTER(gc_problem), ctypes.POINTER(gc_options),
                                           ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.POINTER(gc_stats)])
_sig("gc_rank_to_vector", ctypes.c_int, [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64, _u64p])
_sig("gc_vector_to_rank", ctypes.c_int, [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64, _u64p])
_sig("gc_ranks_to_vectors", ctypes.c_int, [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, _u64p])
_sig("gc_ranks_to_vectors_device", ctypes.c_int, [ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64,
                                                  ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p])
_sig("gc_nccl_id_bytes", ctypes.c_size_t, [])
_sig("gc_nccl_unique_id", ctypes.c_int, [_u8p, ctypes.c_size_t])
_sig("gc_comm_create", ctypes.c_int, [_u8p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_void_p)])
_sig("gc_comm_destroy", ctypes.c_int, [ctypes.c_void_p])
_sig("gc_peer_handle_bytes", ctypes.c_size_t, [])
_sig("gc_peer_handles", ctypes.c_int, [_u8p, ctypes.c_size_t])
_sig("gc_comm_attach_peers", ctypes.c_int, [ctypes.c_void_p, _u8p, ctypes.c_size_t])
_sig("gc_generate_rank", ctypes.c_int, [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int,
                                        ctypes.POINTER(gc_options), ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.POINTER(gc_stats)])
_sig("gc_tile_partition", ctypes.c_int, [ctypes.c_uint32, ctypes.c_int, ctypes.c_int, _u32p, _u32p, _u32p])
_sig("gc_analyze", ctypes.c_int, [_u64p, ctypes.c_uint64, ctypes.c_uint32, ctypes.POINTER(gc_analysis)])
_sig("gc_analyze_device", ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p,
                                         ctypes.POINTER(gc_analysis)])
_sig("gc_strerror", ctypes.c_char_p, [ctypes.c_int])
_sig("gc_last_error", ctypes.c_char_p, [])
_sig("gc_abi_version", ctypes.c_int, [])


class GCError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        self.name = _STATUS.get(status, str(status))
        detail = _lib.gc_last_error().decode()
        super().__init__(f"{where}: {self.name} ({_lib.gc_strerror(status).decode()})"
                         + (f": {detail}" if detail else ""))


def _check(rc: int, where: str):
    if rc != 0:
        raise GCError(rc, where)


def ordering_id(ordering) -> int:
    if isinstance(ordering, str):
        return ORDERINGS[ordering]
    return int(ordering)


def _opts(options) -> gc_options | None:
    if options is None:
        return None
    if isinstance(options, gc_options):
        return options
    o = gc_options()
    o.struct_size = ctypes.sizeof(gc_options)
    for k, v in dict(options).items():
        setattr(o, k, int(v))
    return o


def _ref(o):
    return ctypes.byref(o) if o is not None else None


def _stream_ptr(stream) -> int | None:
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)   # torch.cuda.Stream


# ------------------------------------------------------------------ ABI calls

def gc_strerror(status: int) -> str:
    return _lib.gc_strerror(status).decode()


def gc_last_error() -> str:
    return _lib.gc_last_error().decode()


def gc_abi_version() -> int:
    return _lib.gc_abi_version()


def gc_capacity_bound(n: int, d: int) -> int:
    return int(_lib.gc_capacity_bound(n, d))


def gc_generate(n: int, d: int, ordering="lex", capacity: int | None = None) -> np.ndarray:
    """The greedy code (uint64 array, acceptance order) -- gc_generate()."""
    cap = gc_capacity_bound(n, d) if capacity is None else capacity
    out = np.empty(max(cap, 1), dtype=np.uint64)
    cnt = ctypes.c_uint64(cap)
    _check(_lib.gc_generate(n, d, ordering_id(ordering), out.ctypes.data_as(_u64p), ctypes.byref(cnt)),
           "gc_generate")
    return out[: cnt.value]


def gc_generate_ex(n: int, d: int, ordering="lex", options=None, capacity: int | None = None):
    """(codewords uint64 array, stats dict) -- gc_generate_ex()."""
    cap = gc_capacity_bound(n, d) if capacity is None else capacity
    out = np.empty(max(cap, 1), dtype=np.uint64)
    cnt = ctypes.c_uint64(cap)
    st = gc_stats()
    st.struct_size = ctypes.sizeof(gc_stats)
    o = _opts(options)
    _check(_lib.gc_generate_ex(n, d, ordering_id(ordering), _ref(o), out.ctypes.data_as(_u64p),
                               ctypes.byref(cnt), ctypes.byref(st)), "gc_generate_ex")
    return out[: cnt.value], st.to_dict()


def gc_generate_device(n: int, d: int, ordering, codebook, count, stream=None, options=None,
                       stats: bool = False):
    """Device variant: `codebook` = CUDA tensor of >= capacity 32-bit words, `count` = CUDA
    tensor holding one 64-bit word.  Returns the stats dict if stats=True, else None."""
    o = _opts(options)
    st = None
    if stats:
        st = gc_stats()
        st.struct_size = ctypes.sizeof(gc_stats)
    cap = codebook.numel() * codebook.element_size() // 4
    _check(_lib.gc_generate_device(n, d, ordering_id(ordering), _ref(o), codebook.data_ptr(), cap,
                                   count.data_ptr(), _stream_ptr(stream), _ref(st)), "gc_generate_device")
    return st.to_dict() if st is not None else None


def _problem(n, d, ordering="lex", basis=None, constant_weight=-1, self_orthogonal=False):
    p = gc_problem()
    p.struct_size = ctypes.sizeof(gc_problem)
    p.n, p.d = n, d
    keep = None
    if basis is not None:
        if len(basis) != n:
            raise ValueError(f"a B-ordering basis needs exactly n = {n} vectors, got {len(basis)}")
        keep = (ctypes.c_uint64 * len(basis))(*[int(x) for x in basis])
        p.basis = ctypes.cast(keep, ctypes.POINTER(ctypes.c_uint64))
        p.ordering = GC_B_ORDERING
    else:
        p.ordering = ordering_id(ordering)
    p.constant_weight = int(constant_weight)
    p.self_orthogonal = int(bool(self_orthogonal))
    return p, keep


def gc_construct(n: int, d: int, ordering="lex", basis=None, constant_weight=-1, self_orthogonal=False,
                 options=None, capacity: int | None = None):
    """Generalised construction (B-ordering basis, constant weight, self-orthogonal) --
    gc_construct().  Returns (codewords uint64 array, stats dict)."""
    prob, keep = _problem(n, d, ordering, basis, constant_weight, self_orthogonal)
    if capacity is not None:
        cap = capacity
    elif n > 32 and constant_weight >= 0:        # 64-bit constant-weight path: at most the weight class
        from math import comb
        cap = min(comb(n, constant_weight), 1 << 27)
    else:
        cap = gc_capacity_bound(n, d)
    out = np.empty(max(cap, 1), dtype=np.uint64)
    cnt = ctypes.c_uint64(cap)
    st = gc_stats()
    st.struct_size = ctypes.sizeof(gc_stats)
    o = _opts(options)
    _check(_lib.gc_construct(ctypes.byref(prob), _ref(o), out.ctypes.data_as(_u64p), ctypes.byref(cnt),
                             ctypes.byref(st)), "gc_construct")
    del keep
    return out[: cnt.value], st.to_dict()


def gc_construct_device(n: int, d: int, codebook, count, ordering="lex", basis=None, constant_weight=-1,
                        self_orthogonal=False, stream=None, options=None, stats: bool = False):
    prob, keep = _problem(n, d, ordering, basis, constant_weight, self_orthogonal)
    o = _opts(options)
    st = None
    if stats:
        st = gc_stats()
        st.struct_size = ctypes.sizeof(gc_stats)
    cap = codebook.numel() * codebook.element_size() // 4
    _check(_lib.gc_construct_device(ctypes.byref(prob), _ref(o), codebook.data_ptr(), cap, count.data_ptr(),
                                    _stream_ptr(stream), _ref(st)), "gc_construct_device")
    del keep
    return st.to_dict() if st is not None else None


def gc_analyze(words, pairwise: bool = False, orthogonality: bool = False) -> dict:
    """Code analysis on the GPU (gc_analyze): weight distribution, GF(2) rank, linearity,
    minimum distance (pairwise or, for linear codes, min nonzero weight), self-orthogonality."""
    w = np.ascontiguousarray(np.asarray(words, dtype=np.uint64))
    a = gc_analysis()
    a.struct_size = ctypes.sizeof(gc_analysis)
    flags = (GC_ANALYZE_PAIRWISE if pairwise else 0) | (GC_ANALYZE_ORTHOGONALITY if orthogonality else 0)
    _check(_lib.gc_analyze(w.ctypes.data_as(_u64p) if len(w) else None, len(w), flags, ctypes.byref(a)),
           "gc_analyze")
    return a.to_dict()


def gc_analyze_device(words, M: int | None = None, pairwise: bool = False, orthogonality: bool = False,
                      stream=None) -> dict:
    """As gc_analyze for a CUDA tensor of 32-bit words."""
    a = gc_analysis()
    a.struct_size = ctypes.sizeof(gc_analysis)
    M = words.numel() * words.element_size() // 4 if M is None else M
    flags = (GC_ANALYZE_PAIRWISE if pairwise else 0) | (GC_ANALYZE_ORTHOGONALITY if orthogonality else 0)
    _check(_lib.gc_analyze_device(words.data_ptr() if M else None, M, flags, _stream_ptr(stream), ctypes.byref(a)),
           "gc_analyze_device")
    return a.to_dict()


def gc_rank_to_vector(ordering, n: int, rank: int) -> int:
    v = ctypes.c_uint64()
    _check(_lib.gc_rank_to_vector(ordering_id(ordering), n, rank, ctypes.byref(v)), "gc_rank_to_vector")
    return v.value


def gc_vector_to_rank(ordering, n: int, vec: int) -> int:
    r = ctypes.c_uint64()
    _check(_lib.gc_vector_to_rank(ordering_id(ordering), n, vec, ctypes.byref(r)), "gc_vector_to_rank")
    return r.value


def gc_ranks_to_vectors(ordering, n: int, first: int, count: int) -> np.ndarray:
    out = np.zeros(max(count, 1), dtype=np.uint64)
    _check(_lib.gc_ranks_to_vectors(ordering_id(ordering), n, first, count, out.ctypes.data_as(_u64p)),
           "gc_ranks_to_vectors")
    return out[:count]


def gc_ranks_to_vectors_device(ordering, n: int, first: int, count: int, out, stream=None):
    """Fill the CUDA tensor `out` (>= count 32-bit words) with the device generator's vectors."""
    _check(_lib.gc_ranks_to_vectors_device(ordering_id(ordering), n, first, count, out.data_ptr(),
                                           _stream_ptr(stream)), "gc_ranks_to_vectors_device")
    return out


def gc_tile_partition(K: int, world: int, rank: int) -> tuple[int, int, int]:
    """(part_lo, part_len, Kpad) of `rank` inside a tile of K candidates."""
    lo, ln, kp = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
    _check(_lib.gc_tile_partition(K, world, rank, ctypes.byref(lo), ctypes.byref(ln), ctypes.byref(kp)),
           "gc_tile_partition")
    return lo.value, ln.value, kp.value


def gc_nccl_id_bytes() -> int:
    return int(_lib.gc_nccl_id_bytes())


def gc_nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(_lib.gc_nccl_unique_id(buf, 128), "gc_nccl_unique_id")
    return bytes(buf)


class GcComm:
    """Owns a gc_comm* (gc_comm_create / gc_comm_destroy)."""

    def __init__(self, handle: int, rank: int, world: int):
        self.handle, self.rank, self.world = handle, rank, world

    def close(self):
        if self.handle:
            _lib.gc_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gc_comm_create(nccl_id: bytes | None, rank: int, world: int) -> GcComm:
    h = ctypes.c_void_p()
    if nccl_id is not None:
        idbuf = (ctypes.c_uint8 * len(nccl_id)).from_buffer_copy(nccl_id)
        idlen = len(nccl_id)
    else:
        idbuf, idlen = None, 0
    _check(_lib.gc_comm_create(idbuf, idlen, rank, world, ctypes.byref(h)), "gc_comm_create")
    return GcComm(h.value, rank, world)


def gc_comm_destroy(comm: GcComm):
    comm.close()


def gc_peer_handle_bytes() -> int:
    return int(_lib.gc_peer_handle_bytes())


def gc_peer_handles() -> bytes:
    """CUDA IPC handles of this process's tile-exchange buffers on the current device."""
    nb = gc_peer_handle_bytes()
    buf = (ctypes.c_uint8 * nb)()
    _check(_lib.gc_peer_handles(buf, nb), "gc_peer_handles")
    return bytes(buf)


def gc_comm_attach_peers(comm: GcComm, all_handles: bytes):
    """Open every other rank's exchange buffers (all_handles: the ranks' gc_peer_handles, in rank order)."""
    nb = gc_peer_handle_bytes()
    if len(all_handles) != nb * comm.world:
        raise ValueError(f"expected {comm.world} x {nb} bytes of handles, got {len(all_handles)}")
    buf = (ctypes.c_uint8 * len(all_handles)).from_buffer_copy(all_handles)
    _check(_lib.gc_comm_attach_peers(comm.handle, buf, nb), "gc_comm_attach_peers")


def gc_generate_rank(n: int, d: int, ordering, comm: GcComm | None, codebook, count, stream=None,
                     options=None) -> dict:
    """One rank of a multi-GPU construction (one process per GPU).  Returns the stats dict."""
    o = _opts(options)
    st = gc_stats()
    st.struct_size = ctypes.sizeof(gc_stats)
    cap = codebook.numel() * codebook.element_size() // 4
    _check(_lib.gc_generate_rank(n, d, ordering_id(ordering), _ref(o), comm.handle if comm else None,
                                 codebook.data_ptr(), cap, count.data_ptr(), _stream_ptr(stream),
                                 ctypes.byref(st)), "gc_generate_rank")
    return st.to_dict()


def exported_symbols() -> list[str]:
    """Every function include/gc.h declares (parsed from the header)."""
    txt = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(gc_\w+)\s*\(", txt, re.M)))
