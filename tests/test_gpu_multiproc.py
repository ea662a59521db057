"""The row-sharded path across processes on ONE GPU (the gpurun box has one B200): 2 and 4 ranks,
each a process with its own CUDA context on device 0, exchange CUDA-IPC handles through a gloo
process group and run qp_layer_shard + qp_linear_fwd_sharded_p2p (the fused all-gather epilogue:
peer stores into every rank's y_full, per-rank completion flags, the round-entry barrier and the
wait kernel). Every rank's gathered y_full must equal the float64 oracle on the full layer
(2e-3 normwise), over repeated rounds (eager and CUDA-graph replays) with y_full reused every
round. Also qp_gather_permute (the [P][B][m] -> [B][P*m] step after ncclAllGather) at P = 2/4/8.

NCCL itself refuses two ranks on one device, so qp_linear_fwd_sharded's ncclAllGather runs only at
world 1 here (tests/test_gpu_parity.py); the permutation it applies afterwards is tested below.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
TOL = 2e-3
SEED = 7


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cases, results):
    import torch.distributed as dist
    from oracle import linear
    from paper_2509_20214_b200 import _lib as L
    from qp_synth import activations_fp16, channel_scales, random_code_bytes
    from tests import qp_cases as Q
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for ci, (scheme, x4, d_out, d_in, batch, ydt) in enumerate(cases):
            cb = L.Codebook(scheme, x4, Q.load_fp16(scheme, x4), L=16)
            r = L.Rht(SEED, d_in)
            codes = random_code_bytes(Q.code_bytes(d_out, d_in, scheme, x4), 60 + ci)
            s = channel_scales(d_out, d_in)
            full = L.Layer.from_codes(codes, s, d_out, d_in, scheme, x4, cb, r)
            shard = full.shard(rank, world)
            m = d_out // world
            dtype = torch.float32 if ydt == "f32" else torch.float16
            pg = L.PeerGather(world, rank, m, batch, dtype=dtype)
            errs = []
            print(f"[rank {rank}] case {ci} shard ready", flush=True)
            st = torch.cuda.Stream()
            for rnd in range(3):
                # a different input every round: stale data from the previous round would show
                x = activations_fp16(batch, d_in, seed=100 + rnd)
                ref = linear.linear_from_codes(codes, d_out, d_in, scheme, x4, Q.oracle_codebook(scheme, x4), s,
                                               x.astype(np.float64), SEED)
                xg = torch.from_numpy(x).cuda()
                with torch.cuda.stream(st):
                    pg.forward(shard, xg, stream=st)
                    yh = pg.y.float().cpu().numpy()            # the reader of this round (same stream)
                errs.append(float(np.max(linear.normwise_error(yh, ref))))
                print(f"[rank {rank}] case {ci} round {rnd} err {errs[-1]:.2e}", flush=True)
            # CUDA graph of one round, replayed with the input changing in place
            x = activations_fp16(batch, d_in, seed=200)
            xg = torch.from_numpy(x).cuda()
            with torch.cuda.stream(st):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    pg.forward(shard, xg, stream=st)
                for rep in range(3):
                    xn = activations_fp16(batch, d_in, seed=300 + rep)
                    xg.copy_(torch.from_numpy(xn))
                    g.replay()
                    yh = pg.y.float().cpu().numpy()
                    ref = linear.linear_from_codes(codes, d_out, d_in, scheme, x4, Q.oracle_codebook(scheme, x4), s,
                                                   xn.astype(np.float64), SEED)
                    errs.append(float(np.max(linear.normwise_error(yh, ref))))
            torch.cuda.synchronize()
            dist.barrier()
            results[(rank, ci)] = max(errs)
            pg.close()
            del pg, shard, full
            torch.cuda.synchronize()
            dist.barrier()
    except Exception as e:                       # report, do not hang the other ranks
        results[(rank, -1)] = repr(e)
        raise
    finally:
        dist.destroy_process_group()


CASES = [("tcq", 10, 512, 1024, 1, "f32"), ("vq", 12, 256, 512, 3, "f16"), ("half_tcq", 13, 1024, 1024, 8, "f32")]


@pytest.mark.parametrize("world", [2, 4])
def test_p2p_allgather_across_processes(world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), CASES, results), nprocs=world, join=True)
    errs = dict(results)
    assert all(k[1] >= 0 for k in errs), errs
    assert len(errs) == world * len(CASES), errs
    assert max(errs.values()) <= TOL, errs


def _mworker(rank, world, port, specs, batch, ydt, results):
    """The engine with the fused all-gather (qp_multi_fwd_sharded_p2p): this rank's row shards of
    several layers in one qp_multi; every rank's y_full of every layer against the oracle."""
    import torch.distributed as dist
    from oracle import linear
    from paper_2509_20214_b200 import _lib as L
    from qp_synth import activations_fp16, channel_scales, random_code_bytes
    from tests import qp_cases as Q
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full, codes, scales, shards = [], [], [], []
        cbs = {}
        for li, (d_out, d_in, scheme, x4) in enumerate(specs):
            if (scheme, x4) not in cbs:
                cbs[(scheme, x4)] = L.Codebook(scheme, x4, Q.load_fp16(scheme, x4), L=16)
            c = random_code_bytes(Q.code_bytes(d_out, d_in, scheme, x4), 500 + li)
            s = channel_scales(d_out, d_in)
            f = L.Layer.from_codes(c, s, d_out, d_in, scheme, x4, cbs[(scheme, x4)], L.Rht(SEED, d_in))
            full.append(f)
            codes.append(c)
            scales.append(s)
            shards.append(f.shard(rank, world))
        m = L.Multi(shards)
        assert m.n_engine_launches == m.n_launches
        dtype = torch.float32 if ydt == "f32" else torch.float16
        pg = L.MultiPeerGather(world, rank, [d_out // world for d_out, _, _, _ in specs], batch, dtype=dtype)
        st = torch.cuda.Stream()
        errs = []

        def check(xs_np):
            for li, ((d_out, d_in, scheme, x4), x) in enumerate(zip(specs, xs_np)):
                ref = linear.linear_from_codes(codes[li], d_out, d_in, scheme, x4, Q.oracle_codebook(scheme, x4),
                                               scales[li], x.astype(np.float64), SEED)
                errs.append(float(np.max(linear.normwise_error(pg.ys[li].float().cpu().numpy(), ref))))

        for rnd in range(3):
            xs_np = [activations_fp16(batch, sp[1], seed=700 + 10 * rnd + li) for li, sp in enumerate(specs)]
            xs = [torch.from_numpy(x).cuda() for x in xs_np]
            with torch.cuda.stream(st):
                pg.forward(m, xs, stream=st)
                st.synchronize()
            check(xs_np)
        xs = [torch.empty(batch, sp[1], dtype=torch.float16, device="cuda") for sp in specs]
        with torch.cuda.stream(st):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                pg.forward(m, xs, stream=st)
            for rep in range(3):
                xs_np = [activations_fp16(batch, sp[1], seed=800 + 10 * rep + li) for li, sp in enumerate(specs)]
                for x, xn in zip(xs, xs_np):
                    x.copy_(torch.from_numpy(xn))
                g.replay()
                st.synchronize()
                check(xs_np)
        torch.cuda.synchronize()
        dist.barrier()
        results[rank] = max(errs)
        pg.close()
        del pg, m, shards, full
        torch.cuda.synchronize()
        dist.barrier()
    except Exception as e:
        results[-1 - rank] = repr(e)
        raise
    finally:
        dist.destroy_process_group()


MSPECS = [(512, 1024, "tcq", 10), (256, 1536, "half_tcq", 13), (1024, 512, "tcq", 16), (256, 14336, "tcq", 14)]


@pytest.mark.parametrize("world,batch,ydt", [(2, 1, "f32"), (2, 8, "f16"), (4, 3, "f32"), (4, 1, "f16")])
def test_engine_p2p_allgather_across_processes(world, batch, ydt):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_mworker, args=(world, _free_port(), MSPECS, batch, ydt, results), nprocs=world, join=True)
    errs = dict(results)
    assert sorted(errs) == list(range(world)), errs
    assert max(errs.values()) <= TOL, errs


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("batch", [1, 3, 8])
def test_gather_permute(world, batch):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2509_20214_b200 import _lib as L
    m = 96
    for dtype in (torch.float32, torch.float16):
        src = torch.randn(world, batch, m, device="cuda").to(dtype)
        dst = torch.empty(batch, world * m, dtype=dtype, device="cuda")
        L.gather_permute(src, dst, world, batch, m)
        torch.cuda.synchronize()
        assert torch.equal(dst, src.permute(1, 0, 2).reshape(batch, world * m))


def _kworker(rank, world, port, cases, results):
    """K (column) shards: each rank computes its partial y on the GPU from its columns of x, the
    partials are summed with gloo (NCCL refuses two ranks on one device), the sum must equal the
    oracle's y of the full layer."""
    import torch.distributed as dist
    from oracle import decode, rht
    from paper_2509_20214_b200 import _lib as L
    from qp_synth import activations_fp16, channel_scales, random_code_bytes
    from tests import qp_cases as Q
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for ci, (scheme, x4, d_out, d_in, block, batch) in enumerate(cases):
            cb = L.Codebook(scheme, x4, Q.load_fp16(scheme, x4), L=16)
            r = L.Rht(SEED, d_in, block)
            codes = random_code_bytes(Q.code_bytes(d_out, d_in, scheme, x4), 80 + ci)
            s = channel_scales(d_out, d_in)
            full = L.Layer.from_codes(codes, s, d_out, d_in, scheme, x4, cb, r)
            shard = full.shard_k(rank, world)
            dl = d_in // world
            x = activations_fp16(batch, d_in, seed=90 + ci)
            xg = torch.from_numpy(np.ascontiguousarray(x[:, rank * dl:(rank + 1) * dl])).cuda()
            y = torch.empty(batch, d_out, device="cuda")
            shard.forward(xg, batch, y)
            torch.cuda.synchronize()
            yc = y.cpu().double()
            dist.all_reduce(yc)
            W = decode.decode_layer(codes, d_out, d_in, scheme, x4, Q.oracle_codebook(scheme, x4))
            ref = (rht.rht_apply(x.astype(np.float64), SEED, block) @ W.T) * s.astype(np.float64)[None, :]
            err = float(np.max(np.max(np.abs(yc.numpy() - ref), axis=1) / np.max(np.abs(ref), axis=1)))
            results[(rank, ci)] = err
            del shard, full
    except Exception as e:
        results[(rank, -1)] = repr(e)
        raise
    finally:
        dist.destroy_process_group()


KCASES = {2: [("tcq", 10, 64, 1024, 256, 1), ("vq", 12, 96, 2048, 512, 3)],
          3: [("nuq", 16, 64, 1536, 512, 2)],
          4: [("tcq", 16, 32, 2048, 256, 8)]}


@pytest.mark.parametrize("world", [2, 3, 4])
def test_k_shards_across_processes(world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_kworker, args=(world, _free_port(), KCASES[world], results), nprocs=world, join=True)
    errs = dict(results)
    assert all(k[1] >= 0 for k in errs), errs
    assert len(errs) == world * len(KCASES[world]), errs
    assert max(errs.values()) <= TOL, errs


def test_k_shard_errors_and_nccl_world1():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import decode, rht
    from paper_2509_20214_b200 import _lib as L
    from qp_synth import activations_fp16, channel_scales, random_code_bytes
    from tests import qp_cases as Q
    cb = L.Codebook("tcq", 10, Q.load_fp16("tcq", 10), L=16)
    r = L.Rht(SEED, 1024, 1024)
    codes = random_code_bytes(Q.code_bytes(64, 1024, "tcq", 10), 5)
    s = channel_scales(64, 1024)
    full = L.Layer.from_codes(codes, s, 64, 1024, "tcq", 10, cb, r)
    with pytest.raises(L.QPError) as e:                    # 512-column shards of a 1024 rotation block
        full.shard_k(0, 2)
    assert e.value.status == 3
    hcb = L.Codebook("half_tcq", 13, Q.load_fp16("half_tcq", 13), L=16)
    half = L.Layer.from_codes(random_code_bytes(Q.code_bytes(64, 1024, "half_tcq", 13), 6), s, 64, 1024, "half_tcq",
                              13, hcb, L.Rht(SEED, 1024, 256))
    with pytest.raises(L.QPError) as e:
        half.shard_k(0, 2)
    assert e.value.status == 10
    comm = L.NcclComm(L.NcclComm.unique_id(), 1, 0)
    try:
        sh = full.shard_k(0, 1)
        x = activations_fp16(2, 1024)
        y = torch.empty(2, 64, device="cuda")
        sh.forward_ksharded(torch.from_numpy(x).cuda(), 2, y, comm)
        torch.cuda.synchronize()
        W = decode.decode_layer(codes, 64, 1024, "tcq", 10, Q.oracle_codebook("tcq", 10))
        ref = (rht.rht_apply(x.astype(np.float64), SEED, 1024) @ W.T) * s.astype(np.float64)[None, :]
        err = np.max(np.max(np.abs(y.cpu().numpy() - ref), axis=1) / np.max(np.abs(ref), axis=1))
        assert err <= TOL
        with pytest.raises(L.QPError):
            sh.forward_ksharded(torch.from_numpy(x).cuda(), 2, y, comm, flags=L.QP_Y_ACCUMULATE)
    finally:
        comm.close()
