"""Multi-process (world_size 2, gloo, CPU) tests of the N>1 host logic: NCCL-id sharing,
max-over-ranks timing, and the tile partition every rank derives independently (it
must tile [0, Kpad) exactly, in rank order, in whole mask words)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1507_05398_b200 as gc
        from paper_1507_05398_b200 import dist as gdist

        out = {}
        ident = gdist.share_nccl_id()
        out["id"] = ident
        # the peer-handle exchange of the multi-GPU pipelined engine: every rank ends with every
        # rank's blob, in rank order (fake blobs: IPC handles need a GPU)
        nb = gc.gc_peer_handle_bytes()
        out["handles"] = gdist.share_peer_handles(make_handles=lambda: bytes([rank + 1]) * nb)
        out["max"] = gdist.max_over_ranks(10.0 + rank)
        parts = {}
        for K in (1, 7, 32, 33, 64, 256, 4096, 4097, 65536):
            parts[K] = gc.gc_tile_partition(K, world, rank)
        out["parts"] = parts
        # every rank's (lo, len) gathered: must be identical lengths and contiguous
        t = torch.tensor([parts[4097][0], parts[4097][1]], dtype=torch.int64)
        gathered = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, t)
        out["gathered"] = [tuple(g.tolist()) for g in gathered]
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_host_logic():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0]["id"] == res[1]["id"] and len(res[0]["id"]) == 128
    nb = len(res[0]["handles"]) // world
    assert res[0]["handles"] == res[1]["handles"] == bytes([1]) * nb + bytes([2]) * nb
    assert res[0]["max"] == res[1]["max"] == 11.0
    for K, (lo0, ln0, kp0) in res[0]["parts"].items():
        lo1, ln1, kp1 = res[1]["parts"][K]
        assert kp0 == kp1 >= K and kp0 % (32 * world) == 0
        assert ln0 == ln1 == kp0 // world and ln0 % 32 == 0
        assert lo0 == 0 and lo1 == ln0                 # rank order, contiguous, disjoint
    assert res[0]["gathered"] == res[1]["gathered"]
    assert [g[0] for g in res[0]["gathered"]] == [0, res[0]["gathered"][0][1]]


@pytest.mark.parametrize("world", [1, 2, 4, 8, 64])
def test_partition_covers_tile(world):
    import paper_1507_05398_b200 as gc
    for K in (1, 31, 32, 100, 4096, 8191, 65536):
        covered = []
        for r in range(world):
            lo, ln, kp = gc.gc_tile_partition(K, world, r)
            covered.extend(range(lo, lo + ln))
            assert lo % 32 == 0 and ln % 32 == 0
        assert covered == list(range(kp)) and kp >= K and kp - K < 32 * world


def test_partition_rejects_bad_args():
    import paper_1507_05398_b200 as gc
    for world, rank in ((3, 0), (2, 2), (0, 0), (128, 0), (2, -1)):
        with pytest.raises(gc.GCError):
            gc.gc_tile_partition(64, world, rank)


# ---------------------------------------------------------------------------------------------
# The multi-rank tile-exchange protocol of the pipelined engine (gc_pipeline.cu: q_push,
# q_peers_in, q_flag_empty, the ring depth rule in pipeline_run), modelled with world_size-2
# processes: "peer memory" is a shared-memory tensor every process can store into, the way a rank
# stores into its peers' rings over NVLink.  Every rank screens its partition of tile i (whole
# mask words, gc_tile_partition), stores those words into EVERY rank's ring slot i % RING, then
# raises its flag (tile + 1) for the slot on every rank; a rank resolves tile i once all flags of
# slot i in its own ring read i + 1, and only then commits it.  A rank publishes tile i + D at
# the commit of tile i, so ranks drift at most 2 D tiles apart and a slot is never rewritten
# while a peer still reads it as long as 2 D < RING (the engine uses D <= 7 with 16 slots).
# Random delays make the ranks drift; both must end with the same sequence of resolved tiles,
# equal to a single-process run.

RING, DEPTH, TILES, K = 16, 7, 120, 256


def _mask_words(tile, lo, ln):
    import numpy as np
    rng = np.random.default_rng(1000 + tile)
    full = rng.integers(0, 2**32, size=K // 32, dtype=np.uint64).astype(np.uint32)
    return full[lo // 32:(lo + ln) // 32]


def _protocol_worker(rank, world, port, q, dead, flags, committed):
    import random
    import time

    import numpy as np
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1507_05398_b200 as gc
        from paper_1507_05398_b200 import dist as gdist

        lo, ln, _ = gc.gc_tile_partition(K, world, rank)
        rnd = random.Random(rank)
        digests = []
        pushed = 0                                  # tiles this rank has screened and pushed
        for i in range(TILES):
            # screen + push every published tile (published = at most DEPTH ahead of the commits)
            while pushed < TILES and pushed <= i + DEPTH:
                t = pushed
                s = t % RING
                # slot reuse rule: tile t - RING must be resolved on every rank first
                while t >= RING and min(int(committed[g]) for g in range(world)) <= t - RING:
                    time.sleep(0.0005)
                time.sleep(rnd.random() * 0.002)
                words = _mask_words(t, lo, ln)
                for g in range(world):               # peer stores, then the flags (after a fence)
                    dead[g, s, lo // 32:(lo + ln) // 32] = __import__("torch").from_numpy(words.astype(np.int64))
                for g in range(world):
                    flags[g, s, rank] = t + 1
                pushed += 1
            s = i % RING
            while any(int(flags[rank, s, g]) != i + 1 for g in range(world)):   # q_peers_in
                time.sleep(0.0005)
            full = dead[rank, s].numpy().astype(np.uint64)
            digests.append(int(np.bitwise_xor.reduce(full * np.uint64(2654435761) + np.uint64(i)) & 0xffffffff))
            committed[rank] = i + 1
            time.sleep(rnd.random() * 0.001)
        q.put((rank, digests, gdist.max_over_ranks(float(len(digests)))))
    finally:
        dist.destroy_process_group()


def test_two_rank_exchange_protocol():
    import numpy as np
    import torch

    world = 2
    assert 2 * DEPTH < RING
    dead = torch.zeros((world, RING, K // 32), dtype=torch.int64).share_memory_()
    flags = torch.zeros((world, RING, world), dtype=torch.int64).share_memory_()
    committed = torch.zeros(world, dtype=torch.int64).share_memory_()
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_protocol_worker, args=(r, world, port, q, dead, flags, committed))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, dg, mx = q.get(timeout=300)
        res[r] = (dg, mx)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = []
    for i in range(TILES):                          # single process: the whole mask of every tile
        full = np.concatenate([_mask_words(i, *gc_part[:2]) for gc_part in
                               [(r * (K // world), K // world) for r in range(world)]]).astype(np.uint64)
        ref.append(int(np.bitwise_xor.reduce(full * np.uint64(2654435761) + np.uint64(i)) & 0xffffffff))
    assert res[0][0] == res[1][0] == ref
    assert res[0][1] == res[1][1] == TILES
