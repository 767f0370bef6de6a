"""CPU-only tests of the C-ABI boundary (no GPU needed): the library loads, exports
every symbol include/gc.h declares, validates arguments before touching CUDA, and
its host-side orderings / capacity bound agree with the oracle and with theory."""
import ctypes
import math

import numpy as np
import pytest

import oracle as O
import paper_1507_05398_b200 as gc
from paper_1507_05398_b200 import _binding as B

ORDERS = ["lex", "gray", "glex", "grlex"]


def test_every_declared_symbol_is_exported():
    syms = gc.exported_symbols()
    assert len(syms) >= 14
    lib = ctypes.CDLL(gc.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert gc.gc_abi_version() == 1


def test_status_strings():
    for s in range(9):
        assert gc.gc_strerror(s) and gc.gc_strerror(s) != "unknown status"
    assert gc.gc_strerror(99) == "unknown status"


@pytest.mark.parametrize("n,d,o,status", [
    (0, 1, 0, "GC_EINVAL"), (5, 0, 0, "GC_EINVAL"), (5, 6, 0, "GC_EINVAL"), (5, 2, 4, "GC_EINVAL"),
    (5, 2, -1, "GC_EINVAL"), (33, 3, 0, "GC_EUNSUPPORTED"), (40, 40, 1, "GC_EUNSUPPORTED"),
])
def test_generate_validates_before_cuda(n, d, o, status):
    with pytest.raises(gc.GCError) as e:
        gc.gc_generate(n, d, o, capacity=16)
    assert e.value.name == status
    with pytest.raises(gc.GCError) as e:
        gc.gc_generate_ex(n, d, o, capacity=16)
    assert e.value.name == status


def test_generate_null_pointers_and_bad_options():
    cnt = ctypes.c_uint64(4)
    assert B._lib.gc_generate(7, 3, 0, None, None) == 1            # out_count NULL
    assert B._lib.gc_generate(7, 3, 0, None, ctypes.byref(cnt)) == 1   # NULL buffer, capacity 4
    for bad in ({"tile_min": 48}, {"tile_min": 16}, {"tile_max": 1 << 21}, {"tile_min": 1024, "tile_max": 512},
                {"window0": 1000}, {"emulate_ranks": 3}, {"flags": 0x80000}, {"struct_size": 4},
                {"pipeline_depth": 17}, {"sub_max": 32}, {"partial_s": 16}, {"split_bits": 33}, {"prep_lead": 16}):
        opts = {"struct_size": ctypes.sizeof(B.gc_options)}
        opts.update(bad)
        with pytest.raises(gc.GCError) as e:
            gc.gc_generate_ex(7, 3, "lex", options=opts)
        assert e.value.name == "GC_EINVAL", bad


def test_generate_without_gpu_reports_cuda_error_not_crash():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(gc.GCError) as e:
        gc.gc_generate(7, 3, "lex")
    assert e.value.name in ("GC_ECUDA", "GC_ENOMEM")


def test_device_entry_points_validate():
    assert B._lib.gc_generate_device(7, 3, 0, None, None, 0, None, None, None) == 1
    assert B._lib.gc_generate_device(7, 8, 0, None, None, 0, None, None, None) == 1
    assert B._lib.gc_generate_device(34, 3, 0, None, None, 0, None, None, None) == 4
    assert B._lib.gc_ranks_to_vectors_device(0, 8, 250, 10, None, None) == 1      # NULL out
    assert B._lib.gc_ranks_to_vectors_device(0, 8, 250, 10, 1, None) == 2         # out of range
    assert B._lib.gc_ranks_to_vectors_device(0, 33, 0, 1, 1, None) == 4
    assert B._lib.gc_ranks_to_vectors_device(7, 8, 0, 1, 1, None) == 1
    # communicator: bad world / rank / id
    h = ctypes.c_void_p()
    assert B._lib.gc_comm_create(None, 0, 0, 3, ctypes.byref(h)) == 1
    assert B._lib.gc_comm_create(None, 0, 2, 2, ctypes.byref(h)) == 1
    assert B._lib.gc_comm_create(None, 0, 0, 2, ctypes.byref(h)) == 1
    assert B._lib.gc_comm_create(None, 0, 0, 1, None) == 1
    c = gc.gc_comm_create(None, 0, 1)          # world 1: no NCCL needed
    assert c.handle
    assert B._lib.gc_generate_rank(7, 8, 0, None, c.handle, 1, 16, 1, None, None) == 1
    assert B._lib.gc_generate_rank(7, 3, 0, None, c.handle, None, 16, 1, None, None) == 1
    gc.gc_comm_destroy(c)
    assert B._lib.gc_comm_destroy(None) == 0


def test_capacity_bound():
    # values from the sphere-packing bound
    assert gc.gc_capacity_bound(28, 3) == 9256395
    assert gc.gc_capacity_bound(26, 4) == 1290555
    assert gc.gc_capacity_bound(24, 8) == 4096
    assert gc.gc_capacity_bound(7, 3) == 16
    assert gc.gc_capacity_bound(5, 1) == 32
    assert gc.gc_capacity_bound(0, 1) == 0 and gc.gc_capacity_bound(5, 6) == 0
    for n in range(1, 15):
        for d in range(1, n + 1):
            for o in ORDERS:
                assert len(O.greedy_ball(n, d, o)) <= gc.gc_capacity_bound(n, d)


@pytest.mark.parametrize("ordering", ORDERS)
@pytest.mark.parametrize("n", [1, 3, 8, 13, 16])
def test_host_orderings_match_oracle_tables(ordering, n):
    t = O.order_table(ordering, n)
    got = gc.gc_ranks_to_vectors(ordering, n, 0, 1 << n)
    assert np.array_equal(got.astype(np.uint32), t)
    for r in range(0, 1 << n, max(1, (1 << n) // 97)):
        v = gc.gc_rank_to_vector(ordering, n, r)
        assert v == t[r]
        assert gc.gc_vector_to_rank(ordering, n, v) == r


@pytest.mark.parametrize("ordering", ORDERS)
def test_host_orderings_large_n_properties(ordering):
    # n beyond the oracle's tables: round trip and the class boundaries fixed by binomials
    for n in (28, 40, 63):
        for r in [0, 1, 2, (1 << n) - 1, (1 << (n - 1)), 12345, (1 << n) // 3]:
            v = gc.gc_rank_to_vector(ordering, n, r)
            assert v < (1 << n)
            assert gc.gc_vector_to_rank(ordering, n, v) == r
        if ordering in ("glex", "grlex"):
            off = 0
            for w in range(n + 1):
                first = gc.gc_rank_to_vector(ordering, n, off)
                last = gc.gc_rank_to_vector(ordering, n, off + math.comb(n, w) - 1)
                lo, hi = (1 << w) - 1, ((1 << w) - 1) << (n - w)
                assert (first, last) == ((lo, hi) if ordering == "glex" else (hi, lo))
                off += math.comb(n, w)


def test_host_ordering_errors():
    with pytest.raises(gc.GCError) as e:
        gc.gc_rank_to_vector("lex", 5, 32)
    assert e.value.name == "GC_ERANGE"
    with pytest.raises(gc.GCError) as e:
        gc.gc_vector_to_rank("gray", 5, 32)
    assert e.value.name == "GC_ERANGE"
    with pytest.raises(gc.GCError) as e:
        gc.gc_ranks_to_vectors("lex", 5, 30, 3)
    assert e.value.name == "GC_ERANGE"
    with pytest.raises(gc.GCError) as e:
        gc.gc_rank_to_vector(9, 5, 1)
    assert e.value.name == "GC_EINVAL"
    with pytest.raises(gc.GCError) as e:
        gc.gc_rank_to_vector("lex", 64, 1)
    assert e.value.name == "GC_EINVAL"


def test_construct_validates_problem():
    for kw, status in [
        (dict(n=5, d=2, basis=[1, 2, 3, 8, 16]), "GC_EINVAL"),          # dependent basis
        (dict(n=5, d=2, basis=[1, 2, 4, 8, 32]), "GC_EINVAL"),          # vector >= 2^n
        (dict(n=5, d=2, basis=[1, 2, 4, 8, 0]), "GC_EINVAL"),           # zero vector
        (dict(n=5, d=2, constant_weight=6), "GC_EINVAL"),
        (dict(n=5, d=2, constant_weight=-2), "GC_EINVAL"),
        (dict(n=5, d=6), "GC_EINVAL"),
        (dict(n=33, d=3), "GC_EUNSUPPORTED"),
    ]:
        with pytest.raises(gc.GCError) as e:
            gc.gc_construct(**kw, capacity=64)
        assert e.value.name == status, kw
    # emulate_ranks cannot carry the extensions
    import torch
    if not torch.cuda.is_available():
        with pytest.raises(gc.GCError) as e:
            gc.gc_construct(8, 3, self_orthogonal=True, options={"emulate_ranks": 2}, capacity=64)
        assert e.value.name in ("GC_EUNSUPPORTED", "GC_ECUDA")


def test_attach_peers_validation():
    # argument checks happen before any CUDA call
    import paper_1507_05398_b200 as gc
    nb = gc.gc_peer_handle_bytes()
    assert nb == 128
    one = gc.gc_comm_create(None, 0, 1)
    try:
        with pytest.raises(gc.GCError) as e:
            gc.gc_comm_attach_peers(one, bytes(nb))
        assert e.value.name == "GC_EUNSUPPORTED"          # a single rank has no peers
        with pytest.raises(ValueError):
            gc.gc_comm_attach_peers(one, bytes(nb + 1))
    finally:
        one.close()
    assert B._lib.gc_comm_attach_peers(None, None, nb) == 1          # GC_EINVAL
    buf = (ctypes.c_uint8 * 8)()
    assert B._lib.gc_peer_handles(buf, 8) == 1                       # too small: GC_EINVAL
