"""GPU parity of the persistent multi-layer engine (qp_multi_fwd) and of the full-size C2 layers.

Bars as tests/test_gpu_parity.py: y within 2e-3 normwise of the float64 oracle (reading R16) on
the same seeded inputs, for every layer of an engine launch; the engine's rotation is bitwise the
rotation kernel's (same operations in the same order), so engine and per-layer outputs agree to
fp32 summation-order noise.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import decode, linear  # noqa: E402
from qp_synth import activations_fp16, channel_scales, random_code_bytes  # noqa: E402

from . import qp_cases as Q  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 2e-3
SEED = 7


def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2509_20214_b200 import _lib as L
    return L


_CB, _RHT = {}, {}


def _cb(scheme, bits_x4, L=16):
    Lb = _lib()
    key = (scheme, bits_x4, L)
    if key not in _CB:
        _CB[key] = (Lb.Codebook(scheme, bits_x4, Q.load_fp16(scheme, bits_x4), L=L), Q.oracle_codebook(scheme, bits_x4, L))
    return _CB[key]


def _rht(d_in):
    Lb = _lib()
    if d_in not in _RHT:
        _RHT[d_in] = Lb.Rht(SEED, d_in)
    return _RHT[d_in]


def _make(specs, first_id=40):
    """specs: [(d_out, d_in, scheme, bits_x4)] -> (layers, codes, scales, oracle codebooks)."""
    Lb = _lib()
    out = []
    for i, (d_out, d_in, scheme, x4) in enumerate(specs):
        cb, ocb = _cb(scheme, x4)
        codes = random_code_bytes(Q.code_bytes(d_out, d_in, scheme, x4), first_id + i)
        s = channel_scales(d_out, d_in)
        out.append((Lb.Layer.from_codes(codes, s, d_out, d_in, scheme, x4, cb, _rht(d_in)), codes, s, ocb, scheme, x4))
    return out


def _ref(item, x):
    lay, codes, s, ocb, scheme, x4 = item
    return linear.linear_from_codes(codes, lay.d_out, lay.d_in, scheme, x4, ocb, s, x.astype(np.float64), SEED)


# several shapes / widths on the tb = 9 table: ragged tile counts, d_in with 1 .. 7 Hadamard blocks
TB9_MIX = [(160, 1536, "tcq", 10), (96, 1024, "half_tcq", 13), (64, 3584, "tcq", 16), (256, 512, "tcq", 12),
           (32, 512, "half_tcq", 11), (128, 14336, "tcq", 14)]


@pytest.mark.parametrize("batch", [1, 3, 8])
@pytest.mark.parametrize("y_dtype", [torch.float32, torch.float16])
def test_engine_tb9_mix_vs_oracle(batch, y_dtype):
    Lb = _lib()
    items = _make(TB9_MIX)
    m = Lb.Multi([it[0] for it in items])
    assert m.n_launches == 1 and m.n_engine_launches == 1
    xs_np = [activations_fp16(batch, it[0].d_in, seed=11 + i) for i, it in enumerate(items)]
    xs = [torch.from_numpy(x).cuda() for x in xs_np]
    ys = [torch.full((batch, it[0].d_out), float("nan"), dtype=y_dtype, device="cuda") for it in items]
    n0 = Lb.launch_count()
    m.forward(xs, batch, ys)
    torch.cuda.synchronize()
    assert Lb.launch_count() - n0 == 1                      # the whole path in one launch
    for it, x, y in zip(items, xs_np, ys):
        err = np.max(linear.normwise_error(y.float().cpu().numpy(), _ref(it, x)))
        assert err <= TOL, (it[0].d_out, it[0].d_in, it[4], it[5], err)


@pytest.mark.parametrize("x_dtype", [torch.bfloat16, torch.float32])
def test_engine_input_dtypes_and_prerotated(x_dtype):
    Lb = _lib()
    items = _make(TB9_MIX[:4], first_id=60)
    m = Lb.Multi([it[0] for it in items])
    batch = 2
    xs_np = [activations_fp16(batch, it[0].d_in, seed=21 + i) for i, it in enumerate(items)]
    xs = [torch.from_numpy(x).to("cuda", x_dtype) for x in xs_np]
    ys = [torch.empty(batch, it[0].d_out, dtype=torch.float32, device="cuda") for it in items]
    m.forward(xs, batch, ys)
    # pre-rotated fp16 x' (qp_rht_apply) through the engine: same outputs up to summation order
    xr = []
    for it, x in zip(items, xs):
        t = torch.empty(batch, it[0].d_in, dtype=torch.float16, device="cuda")
        _rht(it[0].d_in).apply(x, batch, t)
        xr.append(t)
    ys2 = [torch.empty_like(y) for y in ys]
    m.forward(xr, batch, ys2, flags=Lb.QP_X_PREROTATED)
    torch.cuda.synchronize()
    for it, x, y, y2 in zip(items, xs, ys, ys2):
        y_ref = _ref(it, x.float().cpu().numpy())           # the values the kernel received
        assert np.max(linear.normwise_error(y.cpu().numpy(), y_ref)) <= TOL
        assert np.max(linear.normwise_error(y2.cpu().numpy(), y.cpu().numpy())) <= 1e-5


def test_engine_repeated_launches_graph_and_accumulate():
    """Self-cleaning workspace, counters, ready flags and the generation counter across many
    launches (eager and CUDA-graph replays), plus QP_Y_ACCUMULATE and a batch change."""
    Lb = _lib()
    items = _make(TB9_MIX, first_id=80)
    m = Lb.Multi([it[0] for it in items])
    refs = {}
    for batch in (4, 1, 8):
        xs_np = [activations_fp16(batch, it[0].d_in, seed=31 + i) for i, it in enumerate(items)]
        xs = [torch.from_numpy(x).cuda() for x in xs_np]
        ys = [torch.empty(batch, it[0].d_out, dtype=torch.float32, device="cuda") for it in items]
        refs[batch] = [_ref(it, x) for it, x in zip(items, xs_np)]
        for _ in range(3):
            m.forward(xs, batch, ys)
        torch.cuda.synchronize()
        for y, r in zip(ys, refs[batch]):
            assert np.max(linear.normwise_error(y.cpu().numpy(), r)) <= TOL
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            m.forward(xs, batch, ys, stream=s)
            s.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                m.forward(xs, batch, ys, stream=s)
            for _ in range(5):
                g.replay()
        torch.cuda.synchronize()
        for y, r in zip(ys, refs[batch]):
            assert np.max(linear.normwise_error(y.cpu().numpy(), r)) <= TOL
        # accumulate: y = 1 + W x
        for y in ys:
            y.fill_(1.0)
        m.forward(xs, batch, ys, flags=Lb.QP_Y_ACCUMULATE)
        torch.cuda.synchronize()
        for y, r in zip(ys, refs[batch]):
            assert np.max(linear.normwise_error(y.cpu().numpy() - 1.0, r)) <= TOL


def test_engine_independent_launches_overlap_safely():
    """QP_INDEPENDENT: consecutive launches do not wait for each other, only for the previous launch
    of the same qp_multi (entry tickets / exit counts). Two objects alternating (as bench.py's
    replicas) and one object back to back, eager and in a CUDA graph, against the oracle."""
    Lb = _lib()
    objs = []
    for rep in range(2):
        items = _make(TB9_MIX, first_id=180 + 10 * rep)
        m = Lb.Multi([it[0] for it in items])
        xs_np = [activations_fp16(2, it[0].d_in, seed=71 + i + 7 * rep) for i, it in enumerate(items)]
        xs = [torch.from_numpy(x).cuda() for x in xs_np]
        ys = [torch.empty(2, it[0].d_out, dtype=torch.float32, device="cuda") for it in items]
        refs = [_ref(it, x) for it, x in zip(items, xs_np)]
        objs.append((m, xs, ys, refs))
    F = Lb.QP_INDEPENDENT
    for k in range(6):
        m, xs, ys, _ = objs[k % 2]
        m.forward(xs, 2, ys, flags=F)
    m0, xs0, ys0, _ = objs[0]
    for _ in range(4):
        m0.forward(xs0, 2, ys0, flags=F)
    torch.cuda.synchronize()
    for m, xs, ys, refs in objs:
        for y, r in zip(ys, refs):
            assert np.max(linear.normwise_error(y.cpu().numpy(), r)) <= TOL
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for k in range(4):
                m, xs, ys, _ = objs[k % 2]
                m.forward(xs, 2, ys, flags=F, stream=s)
        for _ in range(5):
            g.replay()
        s.synchronize()
    for m, xs, ys, refs in objs:
        for y, r in zip(ys, refs):
            assert np.max(linear.normwise_error(y.cpu().numpy(), r)) <= TOL
    # the dependent default after independent launches on the same objects
    for m, xs, ys, refs in objs:
        m.forward(xs, 2, ys)
    torch.cuda.synchronize()
    for m, xs, ys, refs in objs:
        for y, r in zip(ys, refs):
            assert np.max(linear.normwise_error(y.cpu().numpy(), r)) <= TOL


def test_engine_mixed_tables_and_fallback():
    """Layers of different decode tables split into several launch groups: the engine where a
    variant exists (TCQ tb = 9 twice, VQ-3, NUQ-4), the per-layer path for layers without one
    (UNIF-8 / DEC_SCALAR, TCQ-5.0)."""
    Lb = _lib()
    specs = [(160, 1536, "tcq", 10), (96, 1024, "tcq", 16), (128, 2048, "vq", 12), (64, 1024, "vq", 12),
             (96, 1536, "nuq", 16), (64, 512, "unif", 32), (32, 1024, "tcq", 20), (64, 768, "tcq", 8)]
    items = _make(specs, first_id=100)
    m = Lb.Multi([it[0] for it in items])
    assert m.n_launches == 6 and m.n_engine_launches == 4
    batch = 3
    xs_np = [activations_fp16(batch, it[0].d_in, seed=41 + i) for i, it in enumerate(items)]
    xs = [torch.from_numpy(x).cuda() for x in xs_np]
    ys = [torch.empty(batch, it[0].d_out, dtype=torch.float32, device="cuda") for it in items]
    m.forward(xs, batch, ys)
    m.forward(xs, batch, ys)
    torch.cuda.synchronize()
    for it, x, y in zip(items, xs_np, ys):
        assert np.max(linear.normwise_error(y.cpu().numpy(), _ref(it, x))) <= TOL, (it[4], it[5])


def test_engine_errors():
    Lb = _lib()
    items = _make(TB9_MIX[:2], first_id=120)
    m = Lb.Multi([it[0] for it in items])
    xs = [torch.zeros(1, it[0].d_in, dtype=torch.float16, device="cuda") for it in items]
    ys = [torch.zeros(1, it[0].d_out, dtype=torch.float32, device="cuda") for it in items]
    for flags in (Lb.QP_DETERMINISTIC, Lb.QP_FUSE_RHT):
        with pytest.raises(Lb.QPError) as e:
            m.forward(xs, 1, ys, flags=flags)
        assert e.value.status == 1
    with pytest.raises(Lb.QPError) as e:
        m.forward(xs, 9, ys)
    assert e.value.status == 3
    buf = torch.zeros(1, items[0][0].d_in + 8, dtype=torch.float16, device="cuda")
    with pytest.raises(Lb.QPError) as e:                      # x not 16-byte aligned
        m.forward([buf[:, 1:1 + items[0][0].d_in], xs[1]], 1, ys)
    assert e.value.status == 1


# ---- the C2 workload at full size (BASELINE configs[1]): every output element against the oracle ----
C2 = [(d_out, d_in, s, x4) for d_out, d_in in [(4096, 4096), (14336, 4096), (4096, 14336)]
      for s, x4 in [("tcq", 10), ("half_tcq", 13), ("tcq", 16)]]


@pytest.fixture(scope="module")
def c2_reference():
    """The 9 C2 layers (bench.py's shapes and widths, seeded codes) and their float64 oracle
    outputs for an 8-row activation batch (rows 0..B-1 are the batch-B inputs)."""
    _lib()
    items = _make(C2, first_id=200)
    x8 = [activations_fp16(8, it[0].d_in, seed=51 + i) for i, it in enumerate(items)]
    refs = []
    for it, x in zip(items, x8):
        lay, codes, s, ocb, scheme, x4 = it
        W = decode.decode_layer(codes, lay.d_out, lay.d_in, scheme, x4, ocb)
        refs.append(linear.linear_ref(W, s.astype(np.float64), x.astype(np.float64), SEED))
        del W
    return items, x8, refs


@pytest.mark.parametrize("batch", [1, 8])
def test_c2_full_size_per_layer_path(c2_reference, batch):
    items, x8, refs = c2_reference
    for it, x, r in zip(items, x8, refs):
        xg = torch.from_numpy(np.ascontiguousarray(x[:batch])).cuda()
        y = torch.empty(batch, it[0].d_out, dtype=torch.float32, device="cuda")
        it[0].forward(xg, batch, y)
        torch.cuda.synchronize()
        err = np.max(linear.normwise_error(y.cpu().numpy(), r[:batch]))
        assert err <= TOL, (it[0].d_out, it[0].d_in, it[5], err)


@pytest.mark.parametrize("batch", [1, 8])
@pytest.mark.parametrize("y_dtype", [torch.float32, torch.float16])
def test_c2_full_size_engine(c2_reference, batch, y_dtype):
    Lb = _lib()
    items, x8, refs = c2_reference
    m = Lb.Multi([it[0] for it in items])
    assert m.n_launches == 1
    xs = [torch.from_numpy(np.ascontiguousarray(x[:batch])).cuda() for x in x8]
    ys = [torch.empty(batch, it[0].d_out, dtype=y_dtype, device="cuda") for it in items]
    m.forward(xs, batch, ys)
    m.forward(xs, batch, ys)
    torch.cuda.synchronize()
    for it, y, r in zip(items, ys, refs):
        err = np.max(linear.normwise_error(y.float().cpu().numpy(), r[:batch]))
        assert err <= TOL, (it[0].d_out, it[0].d_in, it[5], err)


@pytest.mark.parametrize("batch", [1, 4])
def test_engine_sharded_nccl_world1(batch):
    """qp_multi_fwd_sharded at world size 1 (one GPU per gpurun box): the engine over the shards,
    one grouped ncclAllGather, the permutation for batch > 1 -- against the oracle."""
    Lb = _lib()
    items = _make(TB9_MIX[:4], first_id=140)
    comm = Lb.NcclComm(Lb.NcclComm.unique_id(), 1, 0)
    try:
        shards = [it[0].shard(0, 1) for it in items]
        m = Lb.Multi(shards)
        xs_np = [activations_fp16(batch, it[0].d_in, seed=61 + i) for i, it in enumerate(items)]
        xs = [torch.from_numpy(x).cuda() for x in xs_np]
        ys = [torch.empty(batch, it[0].d_out, dtype=torch.float32, device="cuda") for it in items]
        for _ in range(2):
            m.forward_sharded(xs, batch, ys, comm)
        torch.cuda.synchronize()
        for it, x, y in zip(items, xs_np, ys):
            assert np.max(linear.normwise_error(y.cpu().numpy(), _ref(it, x))) <= TOL
        with pytest.raises(Lb.QPError):                       # full layers are not shards
            Lb.Multi([it[0] for it in items]).forward_sharded(xs, batch, ys, comm)
    finally:
        comm.close()


def test_activation_range_limit_r20():
    """Reading R20 (x' is fp16, no prescale): |x'_i| <= ||x_block||_1 / sqrt(b) <= sqrt(b) max|x|, so
    rows with max|x| * sqrt(b) < 2^15 never overflow. Pin both sides of the documented limit: such
    rows (a constant row with max|x| * sqrt(b) = 3e4 on a 4096 block; a single spike) are within the
    2e-3 bar; a constant row of 6e4 saturates fp16 in x' and the output is not finite (the
    limitation is real, not silently wrong-but-finite)."""
    Lb = _lib()
    items = _make([(64, 4096, "tcq", 10)], first_id=160)
    m = Lb.Multi([items[0][0]])
    b = 4096
    x = np.full((1, b), 0.0, dtype=np.float64)
    x[0, :] = 30000.0 / np.sqrt(b)            # constant row: |x'_i| <= sqrt(b) max|x| = 3e4 < 2^15
    x16 = x.astype(np.float16)
    y = torch.empty(1, 64, device="cuda")
    m.forward([torch.from_numpy(x16).cuda()], 1, [y])
    torch.cuda.synchronize()
    err = np.max(linear.normwise_error(y.cpu().numpy(), _ref(items[0], x16)))
    assert np.isfinite(y.cpu().numpy()).all() and err <= TOL
    # a spike: all mass in one coordinate of one block -> x' entries = x_0 / sqrt(b); 8x beyond 2^15 * sqrt(b)
    xs = np.zeros((1, b), dtype=np.float16)
    xs[0, 0] = 60000.0
    y2 = torch.empty(1, 64, device="cuda")
    m.forward([torch.from_numpy(xs).cuda()], 1, [y2])
    torch.cuda.synchronize()
    assert np.isfinite(y2.cpu().numpy()).all()           # 60000 / 64 = 937.5: representable, no overflow
    err2 = np.max(linear.normwise_error(y2.cpu().numpy(), _ref(items[0], xs)))
    assert err2 <= TOL
    xo = np.full((1, b), 60000.0, dtype=np.float16)       # sqrt(b) * 6e4 = 3.8e6 >> 65504: x'_0 saturates
    y3 = torch.empty(1, 64, device="cuda")
    m.forward([torch.from_numpy(xo).cuda()], 1, [y3])
    torch.cuda.synchronize()
    assert not np.isfinite(y3.cpu().numpy()).all()


@pytest.mark.parametrize("batch", [1, 5])
def test_engine_p2p_world1_and_errors(batch):
    """qp_multi_fwd_sharded_p2p at world size 1 (the stores go to this rank's own y_full; entry
    barrier, delivery and wait kernel run) against the oracle, repeated; rejected flags / fallback."""
    Lb = _lib()
    items = _make(TB9_MIX[:4], first_id=300)
    shards = [it[0].shard(0, 1) for it in items]
    m = Lb.Multi(shards)
    pg = Lb.MultiPeerGather(1, 0, [it[0].d_out for it in items], batch)
    for rnd in range(3):
        xs_np = [activations_fp16(batch, it[0].d_in, seed=400 + 10 * rnd + i) for i, it in enumerate(items)]
        xs = [torch.from_numpy(x).cuda() for x in xs_np]
        pg.forward(m, xs)
        torch.cuda.synchronize()
        for it, x, y in zip(items, xs_np, pg.ys):
            assert np.max(linear.normwise_error(y.cpu().numpy(), _ref(it, x))) <= TOL
    with pytest.raises(Lb.QPError):
        pg.forward(m, xs, flags=Lb.QP_Y_ACCUMULATE)
    with pytest.raises(Lb.QPError):
        pg.forward(m, xs, flags=Lb.QP_INDEPENDENT)
