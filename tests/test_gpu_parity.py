"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle on the same
seeded inputs.

Bars:
  * decoded weights W_hat (qp_dequantize): bit-exact fp16 for every palette quantizer;
  * y = diag(s) W_hat R x (qp_linear_fwd): per batch row max|y - y*| / max|y*| <= 2e-3
    (north star; fp16 operands, fp32 accumulation vs fp64; reading R16);
  * R x (qp_rht_apply): within one fp16 rounding of the fp64 value.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import decode, layout, linear, rht  # noqa: E402
from qp_synth import activations_fp16, channel_scales, random_code_bytes  # noqa: E402

from . import qp_cases as Q  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 2e-3
SEED = 7


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2509_20214_b200 import _lib as L
    return L


_CB = {}


def _pair(scheme, bits_x4, L=16):
    """(library Codebook, oracle codebook dict) from the same frozen fp16 bytes."""
    Lb = _need_gpu()
    if not Q.have_codebook(scheme, bits_x4):
        pytest.skip(f"codebook {Q.codebook_file(scheme, bits_x4)} not built")
    key = (scheme, bits_x4, L)
    if key not in _CB:
        _CB[key] = (Lb.Codebook(scheme, bits_x4, Q.load_fp16(scheme, bits_x4), L=L),
                    Q.oracle_codebook(scheme, bits_x4, L=L))
    return _CB[key]


_RHT = {}


def _rht(d_in):
    from paper_2509_20214_b200 import _lib as Lb
    if d_in not in _RHT:
        _RHT[d_in] = Lb.Rht(SEED, d_in)
    return _RHT[d_in]


def _layer(scheme, bits_x4, d_out, d_in, L=16, layer_id=0):
    from paper_2509_20214_b200 import _lib as Lb
    cb, ocb = _pair(scheme, bits_x4, L)
    r = _rht(d_in)
    codes = random_code_bytes(Q.code_bytes(d_out, d_in, scheme, bits_x4), layer_id)
    s = channel_scales(d_out, d_in)
    lay = Lb.Layer.from_codes(codes, s, d_out, d_in, scheme, bits_x4, cb, r)
    return lay, codes, s, ocb


def _dequant_gpu(lay):
    W = torch.empty(lay.d_out, lay.d_in, dtype=torch.float16, device="cuda")
    lay.dequantize(W)
    torch.cuda.synchronize()
    return W.cpu().numpy()


@pytest.mark.parametrize("scheme,bits_x4", Q.PALETTE)
def test_dequant_bit_exact_every_quantizer(scheme, bits_x4):
    # 3 row tiles x 4 k tiles: several tiles, warps and CTAs per launch
    d_out, d_in = 96, 1024
    lay, codes, _, ocb = _layer(scheme, bits_x4, d_out, d_in)
    Wg = _dequant_gpu(lay)
    Wo = decode.decode_layer(codes, d_out, d_in, scheme, bits_x4, ocb).astype(np.float16)
    assert np.array_equal(Wg.view(np.uint16), Wo.view(np.uint16))


@pytest.mark.parametrize("scheme,bits_x4", [("tcq", 10), ("half_tcq", 13), ("vq", 12), ("nuq", 16)])
def test_dequant_bit_exact_llama_shape(scheme, bits_x4):
    d_out, d_in = 4096, 4096
    lay, codes, _, ocb = _layer(scheme, bits_x4, d_out, d_in, layer_id=3)
    Wg = _dequant_gpu(lay)
    Wo = decode.decode_layer(codes, d_out, d_in, scheme, bits_x4, ocb).astype(np.float16)
    assert np.array_equal(Wg.view(np.uint16), Wo.view(np.uint16))


def _fwd(lay, x_np, batch, y_dtype=torch.float32, x_dtype=torch.float16, flags=0):
    x = torch.from_numpy(np.ascontiguousarray(x_np)).to("cuda", x_dtype)
    y = torch.empty(batch, lay.d_out, dtype=y_dtype, device="cuda")
    lay.forward(x, batch, y, flags=flags)
    torch.cuda.synchronize()
    return y.float().cpu().numpy()


@pytest.mark.parametrize("scheme,bits_x4", Q.TARGET)
@pytest.mark.parametrize("batch", [1, 3, 8])
def test_linear_parity_palette(scheme, bits_x4, batch):
    # ragged: 5 row tiles x 6 k tiles (30 tiles over the persistent grid)
    d_out, d_in = 160, 1536
    lay, codes, s, ocb = _layer(scheme, bits_x4, d_out, d_in, layer_id=1)
    x = activations_fp16(batch, d_in)
    y = _fwd(lay, x, batch)
    y_ref = linear.linear_from_codes(codes, d_out, d_in, scheme, bits_x4, ocb, s, x.astype(np.float64), SEED)
    assert np.max(linear.normwise_error(y, y_ref)) <= TOL


@pytest.mark.parametrize("d_out,d_in,scheme,bits_x4", [
    (4096, 4096, "tcq", 10), (4096, 4096, "half_tcq", 13), (4096, 4096, "tcq", 16),
    (1024, 14336, "tcq", 10), (512, 28672, "vq", 12), (2048, 8192, "nuq", 16),
])
@pytest.mark.parametrize("batch", [1, 8])
def test_linear_parity_llama_shapes(d_out, d_in, scheme, bits_x4, batch):
    lay, codes, s, ocb = _layer(scheme, bits_x4, d_out, d_in, layer_id=2)
    x = activations_fp16(batch, d_in)
    y = _fwd(lay, x, batch)
    y_ref = linear.linear_from_codes(codes, d_out, d_in, scheme, bits_x4, ocb, s, x.astype(np.float64), SEED)
    assert np.max(linear.normwise_error(y, y_ref)) <= TOL


@pytest.mark.parametrize("d_out,d_in,bits_x4", [(14336, 4096, 10), (4096, 14336, 13), (28672, 8192, 16)])
def test_full_size_sampled_rows(d_out, d_in, bits_x4):
    """BASELINE shapes at full size: GPU y against the oracle on sampled row tiles."""
    scheme = "half_tcq" if bits_x4 % 2 else "tcq"
    lay, codes, s, ocb = _layer(scheme, bits_x4, d_out, d_in, layer_id=5)
    batch = 2
    x = activations_fp16(batch, d_in)
    y = _fwd(lay, x, batch)
    offs, _ = layout.tile_offsets(d_out, d_in, scheme, bits_x4)
    rowtile_bytes = offs[1, 0] if offs.shape[0] > 1 else len(codes)
    xr = rht.rht_apply(x.astype(np.float64), SEED)
    for rt in (0, 1, d_out // 32 // 2, d_out // 32 - 1):
        sub = codes[rt * rowtile_bytes:(rt + 1) * rowtile_bytes]
        W = decode.decode_layer(sub, 32, d_in, scheme, bits_x4, ocb)
        y_ref = (xr @ W.T) * s[rt * 32:(rt + 1) * 32][None, :]
        err = np.max(np.abs(y[:, rt * 32:(rt + 1) * 32] - y_ref)) / np.max(np.abs(y_ref))
        assert err <= 4 * TOL      # normalised by this 32-row slice's max (a stricter base)


def test_rht_kernel_vs_oracle():
    Lb = _need_gpu()
    for d_in in (256, 4096, 14336, 28672, 8192):
        r = Lb.Rht(SEED, d_in)
        x = activations_fp16(3, d_in)
        xg = torch.from_numpy(x).cuda()
        out = torch.empty(3, d_in, dtype=torch.float16, device="cuda")
        r.apply(xg, 3, out)
        torch.cuda.synchronize()
        ref = rht.rht_apply(x.astype(np.float64), SEED)
        got = out.float().cpu().numpy()
        # within one fp16 rounding (relative 2^-11) plus fp32 summation noise
        assert np.all(np.abs(got - ref) <= np.abs(ref) * 2 ** -10 + 1e-6 * np.abs(x).max())


def test_input_dtypes_and_prerotated():
    Lb = _need_gpu()
    lay, codes, s, ocb = _layer("tcq", 10, 96, 768)
    x = activations_fp16(2, 768)
    y_ref = linear.linear_from_codes(codes, 96, 768, "tcq", 10, ocb, s, x.astype(np.float64), SEED)
    for xd in (torch.float16, torch.bfloat16, torch.float32):
        y = _fwd(lay, x, 2, x_dtype=xd)
        assert np.max(linear.normwise_error(y, y_ref)) <= TOL
    y16 = _fwd(lay, x, 2, y_dtype=torch.float16)
    assert np.max(linear.normwise_error(y16, y_ref)) <= TOL
    # QP_X_PREROTATED: feed R x from qp_rht_apply
    r = Lb.Rht(SEED, 768)
    xr = torch.empty(2, 768, dtype=torch.float16, device="cuda")
    r.apply(torch.from_numpy(x).cuda(), 2, xr)
    y2 = torch.empty(2, 96, dtype=torch.float32, device="cuda")
    lay.forward(xr, 2, y2, flags=Lb.QP_X_PREROTATED)
    torch.cuda.synchronize()
    assert np.max(linear.normwise_error(y2.cpu().numpy(), y_ref)) <= TOL


def test_edge_cases_and_errors():
    Lb = _need_gpu()
    # smallest layer: a single tile (32 x 256), batch at the maximum 8
    lay, codes, s, ocb = _layer("vq", 8, 32, 256)
    x = activations_fp16(8, 256)
    y = _fwd(lay, x, 8)
    y_ref = linear.linear_from_codes(codes, 32, 256, "vq", 8, ocb, s, x.astype(np.float64), SEED)
    assert np.max(linear.normwise_error(y, y_ref)) <= TOL
    # repeated launches reuse the self-resetting fixup counters
    for _ in range(3):
        assert np.array_equal(_fwd(lay, x, 8), y)
    xg = torch.from_numpy(x).cuda()
    yg = torch.empty(9, 32, device="cuda")
    for bad in (0, 9):
        with pytest.raises(Lb.QPError) as e:
            lay.forward(xg, bad, yg)
        assert e.value.status == 3
    cb, _ = _pair("vq", 8)
    with pytest.raises(Lb.QPError) as e:
        Lb.Layer.from_codes(np.zeros(10, np.uint8), np.ones(40, np.float32), 40, 256, "vq", 8, cb, Lb.Rht(1, 256))
    assert e.value.status == 3
    with pytest.raises(Lb.QPError) as e:
        Lb.Layer.from_codes(np.zeros(10, np.uint8), np.ones(32, np.float32), 32, 256, "vq", 8, cb, Lb.Rht(1, 256))
    assert e.value.status == 6


def test_deterministic_and_atomic_paths():
    """fp32 y defaults to zero-then-add across CTAs; QP_DETERMINISTIC (and fp16 y) use the
    in-order reduction, which is bitwise reproducible. Both meet the parity bar."""
    Lb = _need_gpu()
    lay, codes, s, ocb = _layer("tcq", 10, 4096, 4096)
    x = activations_fp16(4, 4096)
    y_ref = linear.linear_from_codes(codes, 4096, 4096, "tcq", 10, ocb, s, x.astype(np.float64), SEED)
    y1 = _fwd(lay, x, 4, flags=Lb.QP_DETERMINISTIC)
    y2 = _fwd(lay, x, 4, flags=Lb.QP_DETERMINISTIC)
    assert np.array_equal(y1, y2)
    ya = _fwd(lay, x, 4)
    for y in (y1, ya):
        assert np.max(linear.normwise_error(y, y_ref)) <= TOL
    assert np.max(np.abs(ya - y1)) <= 1e-5 * np.max(np.abs(y1))


def test_fused_group_qkv_and_upgate():
    Lb = _need_gpu()
    for shapes, scheme, bits in ([(128, 512), (64, 512), (64, 512)], "half_tcq", 17),   \
                                ([(448, 1024), (448, 1024)], "tcq", 12):
        layers, refs = [], []
        x = activations_fp16(3, shapes[0][1])
        for i, (do, di) in enumerate(shapes):
            lay, codes, s, ocb = _layer(scheme, bits, do, di, layer_id=10 + i)
            layers.append(lay)
            refs.append(linear.linear_from_codes(codes, do, di, scheme, bits, ocb, s, x.astype(np.float64), SEED))
        g = Lb.Group(layers)
        xg = torch.from_numpy(x).cuda()
        ys = [torch.empty(3, do, device="cuda") for do, _ in shapes]
        g.forward(xg, 3, ys)
        torch.cuda.synchronize()
        for y, ref in zip(ys, refs):
            assert np.max(linear.normwise_error(y.cpu().numpy(), ref)) <= TOL


def test_row_shards_concatenate():
    lay, codes, s, ocb = _layer("tcq", 8, 256, 1024)
    x = activations_fp16(2, 1024)
    y_full = _fwd(lay, x, 2)
    parts = []
    for rank in range(4):
        sh = lay.shard(rank, 4)
        parts.append(_fwd(sh, x, 2))
    y_cat = np.concatenate(parts, axis=1)
    y_ref = linear.linear_from_codes(codes, 256, 1024, "tcq", 8, ocb, s, x.astype(np.float64), SEED)
    assert np.max(linear.normwise_error(y_cat, y_ref)) <= TOL
    assert np.max(np.abs(y_cat - y_full)) <= 1e-5 * np.max(np.abs(y_full))


def test_sharded_forward_nccl_world1():
    Lb = _need_gpu()
    lay, codes, s, ocb = _layer("vq", 12, 256, 512)
    comm = Lb.NcclComm(Lb.NcclComm.unique_id(), 1, 0)
    try:
        for batch in (1, 4):
            x = activations_fp16(batch, 512)
            xg = torch.from_numpy(x).cuda()
            y = torch.empty(batch, 256, device="cuda")
            lay.shard(0, 1).forward_sharded(xg, batch, y, comm)
            torch.cuda.synchronize()
            y_ref = linear.linear_from_codes(codes, 256, 512, "vq", 12, ocb, s, x.astype(np.float64), SEED)
            assert np.max(linear.normwise_error(y.cpu().numpy(), y_ref)) <= TOL
    finally:
        comm.close()


def test_offline_quantizer_c1_matches_oracle():
    """Config C1: 256x256 TCQ-2.0, L=12 (reading R1), W ~ N(0,1) seed 0. The C++ encoder and
    the oracle's rotate-half Viterbi agree by path cost (reading R5); decoding is bit-exact."""
    Lb = _need_gpu()
    from qp_synth import gaussian_weights
    cb, ocb = _pair("tcq", 8, L=12)
    alpha = Q.tcq_alpha("tcq", 8, L=12)                # reading R22 (codebooks/tcq_alpha.json)
    cb.set_scale(alpha)
    W = gaussian_weights(256, 256, seed=0)
    try:
        lay = Lb.Layer.quantize_offline(W.astype(np.float32), "tcq", 8, cb, Lb.Rht(SEED, 256))
    finally:
        cb.set_scale(1.0)
    codes_g, s_g = lay.codes(), lay.scales()
    codes_o, s_o = linear.quantize_offline(W.astype(np.float32).astype(np.float64), "tcq", 8, ocb, SEED, alpha=alpha)
    assert np.allclose(s_g, s_o, rtol=1e-6)
    Wt, _ = linear.gaussianize(W.astype(np.float32).astype(np.float64), SEED, alpha)
    Wg = decode.decode_layer(codes_g, 256, 256, "tcq", 8, ocb)
    Wo = decode.decode_layer(codes_o, 256, 256, "tcq", 8, ocb)
    dg, do = np.sum((Wg - Wt) ** 2), np.sum((Wo - Wt) ** 2)
    assert abs(dg - do) / do < 1e-6
    assert np.mean(codes_g == codes_o) > 0.99
    assert np.array_equal(_dequant_gpu(lay).view(np.uint16), Wg.astype(np.float16).view(np.uint16))
    x = activations_fp16(1, 256)
    y = _fwd(lay, x, 1)
    y_ref = linear.linear_ref(Wg, s_g.astype(np.float64), x.astype(np.float64), SEED)
    assert np.max(linear.normwise_error(y, y_ref)) <= TOL


@pytest.mark.parametrize("scheme,bits_x4", [("nuq", 12), ("vq", 10), ("unif", 16)])
def test_offline_rtn_matches_oracle(scheme, bits_x4):
    Lb = _need_gpu()
    from qp_synth import gaussian_weights
    cb, ocb = _pair(scheme, bits_x4)
    W = gaussian_weights(64, 512, seed=4).astype(np.float32)
    lay = Lb.Layer.quantize_offline(W, scheme, bits_x4, cb, Lb.Rht(SEED, 512))
    codes_o, s_o = linear.quantize_offline(W.astype(np.float64), scheme, bits_x4, ocb, SEED)
    assert np.allclose(lay.scales(), s_o, rtol=1e-6)
    assert np.mean(lay.codes() == codes_o) > 0.99


def test_y_accumulate_flag():
    """QP_Y_ACCUMULATE: y += diag(s) W_hat R x on fp32 y (no zeroing), with and without the
    rotation kernel; rejected for fp16 y and with QP_DETERMINISTIC."""
    Lb = _need_gpu()
    lay, codes, s, ocb = _layer("tcq", 10, 1024, 2048, layer_id=21)
    x = activations_fp16(3, 2048)
    y_ref = linear.linear_from_codes(codes, 1024, 2048, "tcq", 10, ocb, s, x.astype(np.float64), SEED)
    y0 = np.random.default_rng(5).standard_normal((3, 1024)).astype(np.float32)
    xg = torch.from_numpy(x).cuda()
    r = _rht(2048)
    xr = torch.empty(3, 2048, dtype=torch.float16, device="cuda")
    r.apply(xg, 3, xr)
    for xin, fl in ((xg, 0), (xr, Lb.QP_X_PREROTATED)):
        y = torch.from_numpy(y0.copy()).cuda()
        lay.forward(xin, 3, y, flags=fl | Lb.QP_Y_ACCUMULATE)
        torch.cuda.synchronize()
        got = y.cpu().numpy() - y0
        assert np.max(linear.normwise_error(got, y_ref)) <= TOL
    with pytest.raises(Lb.QPError):
        lay.forward(xg, 3, torch.empty(3, 1024, dtype=torch.float16, device="cuda"), flags=Lb.QP_Y_ACCUMULATE)
    with pytest.raises(Lb.QPError):
        lay.forward(xg, 3, torch.empty(3, 1024, device="cuda"), flags=Lb.QP_Y_ACCUMULATE | Lb.QP_DETERMINISTIC)


@pytest.mark.parametrize("d_out,d_in,scheme,bits_x4,batch", [
    (256, 4096, "tcq", 10, 1), (256, 4096, "tcq", 10, 2), (320, 14336, "half_tcq", 13, 1),
    (96, 1536, "vq", 8, 3), (64, 256, "tcq", 16, 8), (128, 28672, "nuq", 16, 1), (96, 2048, "tcq", 16, 4),
])
@pytest.mark.parametrize("x_dtype", [torch.float16, torch.bfloat16, torch.float32])
def test_fused_rotation_path(d_out, d_in, scheme, bits_x4, batch, x_dtype):
    """QP_FUSE_RHT fuses the rotation into the GEMV kernel when x' fits its plan (one launch; y
    zeroed in-kernel); the default is rotation kernel + GEMV. Both meet the oracle bar and agree
    with each other (x' is bitwise the same; only the atomic summation order of split row tiles
    differs)."""
    Lb = _need_gpu()
    lay, codes, s, ocb = _layer(scheme, bits_x4, d_out, d_in, layer_id=21)
    x = activations_fp16(batch, d_in)
    xin = x.astype(np.float64)
    if x_dtype != torch.float16:    # the oracle sees the same (rounded) input values
        xin = torch.from_numpy(x).to(x_dtype).float().numpy().astype(np.float64)
    y_ref = linear.linear_from_codes(codes, d_out, d_in, scheme, bits_x4, ocb, s, xin, SEED)
    n0 = Lb.launch_count()
    y_f = _fwd(lay, x, batch, x_dtype=x_dtype, flags=Lb.QP_FUSE_RHT)
    n_fused = Lb.launch_count() - n0
    n0 = Lb.launch_count()
    y_s = _fwd(lay, x, batch, x_dtype=x_dtype)
    n_sep = Lb.launch_count() - n0
    assert n_sep == 2 and n_fused in (1, 2)
    for y in (y_f, y_s):
        assert np.max(linear.normwise_error(y, y_ref)) <= TOL
    assert np.max(np.abs(y_f - y_s)) <= 1e-5 * np.max(np.abs(y_s))
    # fp16 output (in-order reduction, no zeroing) and y accumulate through the fused path
    y16 = _fwd(lay, x, batch, y_dtype=torch.float16, x_dtype=x_dtype, flags=Lb.QP_FUSE_RHT)
    assert np.max(linear.normwise_error(y16, y_ref)) <= TOL
    xt = torch.from_numpy(x).to("cuda", x_dtype)
    for fl in (Lb.QP_FUSE_RHT, 0):          # (owned row tiles too: 64x256 has one tile per row tile)
        y = torch.full((batch, d_out), 0.25, device="cuda")
        lay.forward(xt, batch, y, flags=fl | Lb.QP_Y_ACCUMULATE)
        lay.forward(xt, batch, y, flags=fl | Lb.QP_Y_ACCUMULATE)
        torch.cuda.synchronize()
        assert np.max(linear.normwise_error(y.cpu().numpy() - 0.25, 2 * y_ref)) <= TOL


def test_fused_rotation_is_single_kernel_at_batch1():
    """With QP_FUSE_RHT the C2 shapes at batch 1 take the one-kernel path; without it, two."""
    Lb = _need_gpu()
    for d_out, d_in in ((4096, 4096), (1024, 14336)):
        lay, _, _, _ = _layer("tcq", 10, d_out, d_in, layer_id=22)
        x = activations_fp16(1, d_in)
        for fl, n in ((Lb.QP_FUSE_RHT, 1), (0, 2)):
            n0 = Lb.launch_count()
            _fwd(lay, x, 1, flags=fl)
            assert Lb.launch_count() - n0 == n


def test_fused_rotation_repeated_launches_in_graph():
    """The in-kernel zeroing barrier is self-resetting: many back-to-back launches (captured in
    a CUDA graph, as the bench runs them) keep producing the same y."""
    Lb = _need_gpu()
    lay, codes, s, ocb = _layer("tcq", 10, 2048, 4096, layer_id=23)
    x = torch.from_numpy(activations_fp16(1, 4096)).cuda()
    y_ref = linear.linear_from_codes(codes, 2048, 4096, "tcq", 10, ocb, s, x.cpu().numpy().astype(np.float64), SEED)
    y = torch.empty(1, 2048, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        lay.forward(x, 1, y, flags=Lb.QP_FUSE_RHT, stream=st)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(16):
                lay.forward(x, 1, y, flags=Lb.QP_FUSE_RHT, stream=st)
        for _ in range(4):
            g.replay()
        st.synchronize()
    assert np.max(linear.normwise_error(y.cpu().numpy(), y_ref)) <= TOL


@pytest.mark.parametrize("scheme,bits_x4", [("nuq", 16), ("vq", 12), ("tcq", 10)])
def test_batch8_row_pair_units_and_groups(scheme, bits_x4):
    """Batch 8 with a small decode table runs row-pair work units (RP = 2): the two row tiles of a
    pair share the x' fragments. Covered on a fused group whose members split row pairs unevenly
    (3 + 1 row tiles) and with fewer units than SMs (the grid shrinks), and on a ragged k range."""
    Lb = _need_gpu()
    shapes = [(96, 768), (32, 768)]
    x = activations_fp16(8, 768)
    layers, refs = [], []
    for i, (do, di) in enumerate(shapes):
        lay, codes, s, ocb = _layer(scheme, bits_x4, do, di, layer_id=30 + i)
        layers.append(lay)
        refs.append(linear.linear_from_codes(codes, do, di, scheme, bits_x4, ocb, s, x.astype(np.float64), SEED))
    g = Lb.Group(layers)
    ys = [torch.empty(8, do, device="cuda") for do, _ in shapes]
    g.forward(torch.from_numpy(x).cuda(), 8, ys)
    torch.cuda.synchronize()
    for y, ref in zip(ys, refs):
        assert np.max(linear.normwise_error(y.cpu().numpy(), ref)) <= TOL
    lay, codes, s, ocb = _layer(scheme, bits_x4, 1024, 2560, layer_id=33)
    x = activations_fp16(8, 2560)
    y = _fwd(lay, x, 8)
    ref = linear.linear_from_codes(codes, 1024, 2560, scheme, bits_x4, ocb, s, x.astype(np.float64), SEED)
    assert np.max(linear.normwise_error(y, ref)) <= TOL


@pytest.mark.parametrize("d_out,d_in,scheme,bits_x4,L", [
    (256, 256, "tcq", 8, 12),        # config C1
    (32, 512, "tcq", 10, 16),        # TCQ-2.5, L = 16: 1 x 2 tiles = 64 trellises
    (32, 512, "half_tcq", 13, 16),   # half-TCQ 3.25: k tile 0 at s = 6, k tile 1 at s = 7
])
def test_gpu_trellis_encoder_matches_host_and_oracle(d_out, d_in, scheme, bits_x4, L):
    """qp_quantize_offline_gpu (NEXT-1): the rotate-half Viterbi on the GPU, float64 in the host
    encoder's operation order, yields bitwise the host encoder's codes; its total distortion equals
    the oracle's rotate-half encoder's (path cost, reading R5)."""
    Lb = _need_gpu()
    from qp_synth import gaussian_weights
    cb, ocb = _pair(scheme, bits_x4, L=L)
    alpha = Q.tcq_alpha(scheme, bits_x4, L=L)           # reading R22
    W = gaussian_weights(d_out, d_in, seed=0).astype(np.float32)
    r = Lb.Rht(SEED, d_in)
    cb.set_scale(alpha)
    try:
        lay_g = Lb.Layer.quantize_offline(W, scheme, bits_x4, cb, r, gpu=True)
        lay_h = Lb.Layer.quantize_offline(W, scheme, bits_x4, cb, r)
    finally:
        cb.set_scale(1.0)
    codes_g, codes_h = lay_g.codes(), lay_h.codes()
    assert np.array_equal(codes_g, codes_h)
    assert np.array_equal(lay_g.scales(), lay_h.scales())
    Wt, s_o = linear.gaussianize(W.astype(np.float64), SEED, alpha)
    assert np.allclose(lay_g.scales(), s_o, rtol=1e-6)
    codes_o, _ = linear.quantize_offline(W.astype(np.float64), scheme, bits_x4, ocb, SEED, alpha=alpha)
    Wg = decode.decode_layer(codes_g, d_out, d_in, scheme, bits_x4, ocb)
    Wo = decode.decode_layer(codes_o, d_out, d_in, scheme, bits_x4, ocb)
    dg, do = np.sum((Wg - Wt) ** 2), np.sum((Wo - Wt) ** 2)
    assert abs(dg - do) / do < 1e-6


@pytest.mark.parametrize("scheme,bits_x4,tol", [
    ("tcq", 8, 0.02),    # P:909 Ours-TCQ-2 (L = 16, T = 256, tlut_bits = 9, alpha of reading R22)
    ("vq", 8, 0.02),     # P:911 Ours-VQ-2 (our k-means codebook: reading R21)
    ("nuq", 8, 0.005),   # P:910 Ours-NUQ-2
])
def test_table5_distortion_at_scale(scheme, bits_x4, tol):
    """Table 5 at real scale through the product: a 1024x4096 N(0,1) matrix quantized by
    qp_quantize_offline_gpu (TCQ trellis search on the GPU, L = 16), decoded by qp_dequantize;
    the mean squared error against the oracle's standardized weights W~ matches the paper's
    distortion (4 M samples: sampling std ~2e-5)."""
    Lb = _need_gpu()
    from qp_synth import gaussian_weights
    cb, _ = _pair(scheme, bits_x4, L=16)
    alpha = Q.tcq_alpha(scheme, bits_x4)               # reading R22 (1 for VQ / NUQ)
    d_out, d_in = 1024, 4096
    W = gaussian_weights(d_out, d_in, seed=0).astype(np.float32)
    cb.set_scale(alpha)
    try:
        lay = Lb.Layer.quantize_offline(W, scheme, bits_x4, cb, Lb.Rht(SEED, d_in), gpu=True)
    finally:
        cb.set_scale(1.0)
    W_hat = _dequant_gpu(lay).astype(np.float64)
    Wt, s1 = linear.gaussianize(W.astype(np.float64), SEED)
    # reconstruction of the standardized rows: (stored scale / s) * W_hat = alpha * W_hat
    rec = W_hat * (lay.scales().astype(np.float64) / s1)[:, None]
    d = float(np.mean((Wt - rec) ** 2))
    from . import golden_values as G
    paper = G.table5(f"{scheme}-2.0")                 # tests/golden/table5_distortion.json
    assert abs(d - paper) / paper < tol, d
    assert d >= 2.0 ** (-2 * bits_x4 / 4)       # rate-distortion bound


def test_torch_caching_allocator_backs_layers():
    """qp_set_allocator through the binding: a layer allocated from PyTorch's caching allocator
    computes the same y, and its memory shows up in torch's accounting."""
    Lb = _need_gpu()
    _pair("tcq", 10)        # codebook and rotation are cached across tests: create them (and so
    _rht(1024)              # later free them) with the default allocator
    try:
        before = torch.cuda.memory_allocated()
        Lb.use_torch_allocator(True)
        lay, codes, s, ocb = _layer("tcq", 10, 256, 1024, layer_id=40)
        assert torch.cuda.memory_allocated() - before >= lay.code_bytes
        x = activations_fp16(2, 1024)
        y = _fwd(lay, x, 2)
        ref = linear.linear_from_codes(codes, 256, 1024, "tcq", 10, ocb, s, x.astype(np.float64), SEED)
        assert np.max(linear.normwise_error(y, ref)) <= TOL
        del lay
    finally:
        Lb.use_torch_allocator(False)


@pytest.mark.parametrize("batch,y_dtype", [(1, torch.float32), (3, torch.float16), (8, torch.float32)])
def test_fused_allgather_p2p_world1(batch, y_dtype):
    """qp_linear_fwd_sharded_p2p (NEXT-2) at world size 1: the epilogue's direct stores into the
    (here: own) y_full, the grid-completion signal and the wait kernel. Repeated launches and a
    CUDA graph check that the counters self-reset / advance (no host-side epoch)."""
    Lb = _need_gpu()
    lay, codes, s, ocb = _layer("tcq", 10, 1024, 2048, layer_id=41)
    x = activations_fp16(batch, 2048)
    ref = linear.linear_from_codes(codes, 1024, 2048, "tcq", 10, ocb, s, x.astype(np.float64), SEED)
    shard = lay.shard(0, 1)
    pg = Lb.PeerGather(1, 0, 1024, batch, dtype=y_dtype)
    xg = torch.from_numpy(x).cuda()
    for _ in range(3):
        pg.y.zero_()
        pg.forward(shard, xg)
        torch.cuda.synchronize()
        assert np.max(linear.normwise_error(pg.y.float().cpu().numpy(), ref)) <= TOL
    assert int(pg.flags[1].item()) == 3 and int(pg.flags[0].item()) == 3
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            pg.forward(shard, xg, stream=st)
        pg.y.zero_()
        for _ in range(4):
            g.replay()
        st.synchronize()
    assert int(pg.flags[1].item()) == 7
    assert np.max(linear.normwise_error(pg.y.float().cpu().numpy(), ref)) <= TOL


@pytest.mark.parametrize("d_out,d_in,scheme,bits_x4,batch", [
    (4096, 4096, "tcq", 10, 1), (1024, 14336, "half_tcq", 13, 3), (160, 1536, "vq", 12, 8), (512, 2048, "nuq", 16, 2),
])
def test_fp16_output_through_workspace(d_out, d_in, scheme, bits_x4, batch):
    """fp16 y takes the atomic epilogue through the layer's fp32 workspace: split row tiles add into
    it and the warp completing a row tile's k range converts the tile (per-row-tile counters that
    self-reset). Same bar as fp32 y; agrees with the in-order (QP_DETERMINISTIC) fp16 path; stable
    over repeated launches; groups route members' rows."""
    Lb = _need_gpu()
    lay, codes, s, ocb = _layer(scheme, bits_x4, d_out, d_in, layer_id=50)
    x = activations_fp16(batch, d_in)
    ref = linear.linear_from_codes(codes, d_out, d_in, scheme, bits_x4, ocb, s, x.astype(np.float64), SEED)
    ys = [_fwd(lay, x, batch, y_dtype=torch.float16) for _ in range(3)]
    yd = _fwd(lay, x, batch, y_dtype=torch.float16, flags=Lb.QP_DETERMINISTIC)
    for y in ys + [yd]:
        assert np.max(linear.normwise_error(y, ref)) <= TOL
    for y in ys:
        assert np.max(np.abs(y - yd)) <= 2e-3 * np.max(np.abs(yd))
    # fused group with fp16 outputs
    shapes = [(96, 512), (64, 512), (32, 512)]
    xg = activations_fp16(batch, 512)
    layers, refs = [], []
    for i, (do, di) in enumerate(shapes):
        l2, c2, s2, o2 = _layer(scheme, bits_x4, do, di, layer_id=60 + i)
        layers.append(l2)
        refs.append(linear.linear_from_codes(c2, do, di, scheme, bits_x4, o2, s2, xg.astype(np.float64), SEED))
    g = Lb.Group(layers)
    outs = [torch.empty(batch, do, device="cuda", dtype=torch.float16) for do, _ in shapes]
    g.forward(torch.from_numpy(xg).cuda(), batch, outs)
    torch.cuda.synchronize()
    for o, r in zip(outs, refs):
        assert np.max(linear.normwise_error(o.float().cpu().numpy(), r)) <= TOL
