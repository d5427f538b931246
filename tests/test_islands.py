"""Islands (K4): the run_ga block bests are exchanged with one allgather per
generation.  CPU: the torch.distributed adapter (gloo, world_size 2) delivers
records in rank order.  GPU: 1 vs 2 islands (two processes on one device,
gloo exchange -- the kernels never wait on each other) give the identical
RunResult, the reference's worker-count invariance (test_ga.cpp:401-418)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _allgather_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1610_10061_b200 as pm
    fn = pm.torch_allgather()
    send = np.arange(5, dtype=np.uint64) + 100 * rank
    recv = np.zeros(5 * world, dtype=np.uint64)
    rc = fn(send.ctypes.data, send.nbytes, recv.ctypes.data, None)
    q.put((rank, rc, recv.tolist()))
    dist.destroy_process_group()


def test_torch_allgather_adapter_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_allgather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(60)
    want = list(range(5)) + [100 + i for i in range(5)]
    for rank, rc, recv in res:
        assert rc == 0 and recv == want


def _island_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1610_10061_b200 as pm
    from oracle.oracle import Oracle
    o = Oracle()
    costs = o.synth_euclid(300)
    ctx = pm.Context(0)
    ctx.set_instance(costs, 300, 300, 30)
    out = []
    for pop in ("reference", "device"):
        cfg = pm.ga_config(nb=8, nt=32, evolve_limit=5, saturation=5, seed=4, population=pop)
        r = ctx.run_ga(cfg, rank=rank, world=world, allgather=pm.torch_allgather())
        out.append((r["best_cost"], r["best"].tolist(), r["kernels_executed"], r["kernel_of_best"],
                    r["per_kernel_best_costs"].tolist()))
    q.put((rank, out))
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_islands_world_size_invariance():
    import paper_1610_10061_b200 as pm
    from oracle.oracle import Oracle
    o = Oracle()
    costs = o.synth_euclid(300)
    single = []
    with pm.Context(0) as ctx:
        ctx.set_instance(costs, 300, 300, 30)
        for pop in ("reference", "device"):
            r = ctx.run_ga(pm.ga_config(nb=8, nt=32, evolve_limit=5, saturation=5, seed=4, population=pop))
            single.append((r["best_cost"], r["best"].tolist(), r["kernels_executed"], r["kernel_of_best"],
                           r["per_kernel_best_costs"].tolist()))
    c = mp.get_context("spawn")
    q = c.Queue()
    port = _free_port()
    procs = [c.Process(target=_island_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(60)
    for rank, out in res:
        assert out == single, rank


@pytest.mark.gpu
def test_native_nccl_exchange_single_rank():
    """pm_nccl_* (the library's own NCCL island exchange): a one-rank
    communicator returns the record unchanged, and run_ga through it equals the
    plain run.  (Several ranks need several GPUs; the rank-order contract is
    the one the gloo test above checks for the torch adapter.)"""
    import paper_1610_10061_b200 as pm
    from paper_1610_10061_b200 import synth
    comm = pm.NcclComm(pm.nccl_unique_id(), 0, 1, 0)
    data = bytes(range(200)) * 3
    assert comm.allgather(data) == data
    ctx = pm.Context(0)
    ctx.set_instance(synth.euclid_costs(300, 12345), 300, 300, 30)
    cfg = pm.ga_config(nb=4, nt=32, evolve_limit=5, saturation=5, seed=3)
    a = ctx.run_ga(cfg)
    b = ctx.run_ga(cfg, rank=0, world=1, allgather=comm)
    assert a["best_cost"] == b["best_cost"] and (a["best"] == b["best"]).all()
    assert (a["per_kernel_best_costs"] == b["per_kernel_best_costs"]).all()
    comm.close()
    ctx.close()


def _device_ring(world):
    """An in-process stand-in for a device all-gather (pm_allgather_device_fn)
    between `world` contexts on one GPU: each rank copies its device record into
    every rank's device receive buffer (cudaMemcpy, peer-free on one device);
    host barriers order the copies -- no kernel waits on another rank."""
    import threading

    from cuda.bindings import runtime as rt
    bar = threading.Barrier(world)
    recv = [None] * world

    def make(rank):
        def fn(send, nbytes, recv_dev, stream, _user):
            try:
                rt.cudaStreamSynchronize(stream)  # this rank's records are written
                recv[rank] = recv_dev
                bar.wait()
                for r2 in range(world):
                    (err,) = rt.cudaMemcpy(recv[r2] + rank * nbytes, send, nbytes,
                                           rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
                    if err != rt.cudaError_t.cudaSuccess:
                        return 1
                bar.wait()  # every rank's buffer is complete before any step kernel reads it
                return 0
            except Exception:
                return 1
        return fn
    return [make(r) for r in range(world)]


@pytest.mark.gpu
@pytest.mark.parametrize("world,team", [(2, False), (4, False), (2, True)])
def test_device_resident_exchange_matches_one_island(world, team):
    """pm_run_ga_islands_device -- the path the native NCCL exchange takes:
    block records gathered device to device, the generation step (global best,
    stop rule, migration) on the device -- gives the one-island RunResult for
    2 and 4 islands, both migration modes, and both population draws."""
    import threading

    import paper_1610_10061_b200 as pm
    from oracle.oracle import Oracle
    o = Oracle()
    costs = o.synth_euclid(300)
    for pop in ("reference", "device"):
        cfg = dict(nb=8, nt=32, evolve_limit=6, saturation=6, seed=9, population=pop, team=team)
        with pm.Context(0) as ctx:
            ctx.set_instance(costs, 300, 300, 30)
            single = ctx.run_ga(pm.ga_config(**cfg))
        fns = _device_ring(world)
        out = [None] * world

        def run(rank):
            with pm.Context(0) as c:
                c.set_instance(costs, 300, 300, 30)
                out[rank] = c.run_ga(pm.ga_config(**cfg), rank=rank, world=world, allgather_device=fns[rank])

        th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join(300)
        for r in range(world):
            got = out[r]
            assert got is not None, r
            assert got["best_cost"] == single["best_cost"] and (got["best"] == single["best"]).all()
            assert got["kernels_executed"] == single["kernels_executed"]
            assert got["kernel_of_best"] == single["kernel_of_best"]
            assert (got["per_kernel_best_costs"] == single["per_kernel_best_costs"]).all()
