"""Multi-rank window sharding on the CPU: world size 2 over gloo.

The product path runs one process per GPU with NCCL; the host-side logic --
activity-balanced contiguous window shards and the single all-reduce of the
per-net int64 sums -- is exercised here with the CPU oracle standing in for
each rank's GPU shard (test infrastructure only)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2203_06117_b200 import distributed


def test_shards_tile_the_windows_and_balance_activity():
    w = np.array([1, 1, 1, 50, 1, 1, 1, 1, 50, 1], dtype=np.int64)
    for world in (1, 2, 3, 4, 8):
        edges = [distributed.shard_windows(w.size, world, r, w) for r in range(world)]
        assert edges[0][0] == 0 and edges[-1][1] == w.size
        assert all(a[1] == b[0] for a, b in zip(edges, edges[1:]))
    lo, hi = distributed.shard_windows(w.size, 2, 0, w)
    assert 3 <= hi <= 5  # the two heavy windows end up on different ranks
    assert distributed.shard_windows(10, 4, 1) == (2, 5)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import torch.distributed as dist
    import gen
    import paper_2203_06117_b200 as api
    from oracle import port as oport
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    docs = gen.make_docs(31337, n_gates=150, n_pis=6, windows=12, duration_ps=6000,
                         max_toggles=80)
    nl, lv, delays, waves, duration, b, stim = gen.load(docs, api)
    d = oport.Design(lv, delays)
    st = oport.Stimulus(gen.oracle_inputs(nl, waves), b)

    def runner(w_lo, w_hi):
        a = oport.two_pass_simulate(d, st, pct=docs.pct, window_range=(w_lo, w_hi))
        s = oport.compute_stats(d, st, a)
        tot = (int(a["filtered"].sum()), int(a["ic_filtered"].sum()), int(a["discarded"].sum()))
        return s["t1"], s["tc"], s["ig"], tot

    model = api.compile_design(lv, delays)
    (t1, tc, ig, tot), (lo, hi) = distributed.simulate_sharded(model, stim, docs.pct,
                                                               runner=runner)
    q.put((rank, lo, hi, t1, tc, ig, tot))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_allreduce_equals_single_run(oracle_lib):
    import gen
    import paper_2203_06117_b200 as api
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    # shards are contiguous, cover everything, and both ranks hold the sum
    assert res[0][1] == 0 and res[0][2] == res[1][1] and res[1][2] == 12
    assert res[0][2] not in (0, 12)
    docs = gen.make_docs(31337, n_gates=150, n_pis=6, windows=12, duration_ps=6000,
                         max_toggles=80)
    nl, lv, delays, waves, duration, b, stim = gen.load(docs, api)
    _, _, arena, full = oracle_lib.simulate(lv, delays, gen.oracle_inputs(nl, waves), b)
    for r in res:
        assert np.array_equal(r[3], full["t1"]) and np.array_equal(r[4], full["tc"])
        assert np.array_equal(r[5], full["ig"])
        assert r[6] == (int(arena["filtered"].sum()), int(arena["ic_filtered"].sum()),
                        int(arena["discarded"].sum()))


def _gpu_rank(rank, world, port, q):
    # both ranks drive the GPU engine on cuda:0 (one GPU in this pool); they
    # never wait on each other on the device: the sums go through gloo
    import torch.distributed as dist
    import gen
    import paper_2203_06117_b200 as api
    from paper_2203_06117_b200 import synth
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    docs = gen.make_docs(4242, n_gates=400, n_pis=8, windows=40, duration_ps=20_000,
                         max_toggles=300)
    nl, lv, delays, waves, duration, b, stim = gen.load(docs, api)
    model = api.compile_design(lv, delays)
    out.append(distributed.simulate_sharded(model, stim, docs.pct))
    cfg = synth.config("C2", gates=20_000, windows=700)
    m = synth.design(cfg)
    out.append(distributed.simulate_sharded(m, synth.stimulus(cfg, 0, 700), cfg.pct))
    q.put((rank, [((list(map(np.asarray, r[0][:3])), r[0][3]), r[1]) for r in out]))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_two_rank_gpu_runner_equals_single_run():
    import gen
    import paper_2203_06117_b200 as api
    from paper_2203_06117_b200 import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_gpu_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=500) for _ in range(2)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    docs = gen.make_docs(4242, n_gates=400, n_pis=8, windows=40, duration_ps=20_000,
                         max_toggles=300)
    nl, lv, delays, waves, duration, b, stim = gen.load(docs, api)
    single = [api.simulate_stats(api.compile_design(lv, delays), stim,
                                 pathpulse_pct=docs.pct)]
    cfg = synth.config("C2", gates=20_000, windows=700)
    single.append(api.simulate_stats(synth.design(cfg), synth.stimulus(cfg, 0, 700),
                                     pathpulse_pct=cfg.pct))
    for case, ref in enumerate(single):
        shards = [res[r][1][case][1] for r in range(2)]
        assert shards[0][0] == 0 and shards[0][1] == shards[1][0] < shards[1][1]
        for r in range(2):
            (arrs, totals), _ = res[r][1][case]
            for a, x in zip(arrs, ref[:3]):
                assert np.array_equal(a, x)
            assert tuple(totals) == tuple(ref[3])


@pytest.mark.gpu
def test_library_nccl_allreduce_single_rank():
    # gs_nccl_unique_id / gs_nccl_comm_create / gs_allreduce_stats on a
    # one-rank communicator: the in-place int64 sum is the identity, and the
    # sharded runner takes the library's all-reduce path with it
    import torch
    import gen
    import paper_2203_06117_b200 as api
    from paper_2203_06117_b200 import _native
    uid = _native.nccl_unique_id()
    assert len(uid) == _native.NCCL_ID_BYTES
    comm = _native.NcclComm(uid, 1, 0)
    x = torch.arange(-5, 1000, dtype=torch.int64, device="cuda") * 7919
    y = x.clone()
    comm.allreduce_stats(y.data_ptr(), y.numel(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(x, y)
    docs = gen.make_docs(4242, n_gates=400, n_pis=8, windows=40, duration_ps=20_000,
                         max_toggles=300)
    nl, lv, delays, waves, duration, b, stim = gen.load(docs, api)
    model = api.compile_design(lv, delays)
    (t1, tc, ig, tot), _ = distributed.simulate_sharded(model, stim, docs.pct, comm=comm)
    ref = api.simulate_stats(model, stim, pathpulse_pct=docs.pct)
    assert np.array_equal(t1, ref[0]) and np.array_equal(tc, ref[1]) and tot == ref[3]
