"""ctypes binding of libqpalette.so (include/qpalette.h): argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module only converts
Python objects (torch tensors for device memory, numpy arrays for host memory) into the
pointers and sizes of the C ABI. If the shared library is missing it raises -- there is
no Python or CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libqpalette.so")
LIB_PATH = os.environ.get("QP_LIB_PATH", LIB_PATH)   # experiments: an alternative in-tree build

QP_OK = 0
STATUS = {0: "QP_OK", 1: "QP_ERR_INVALID_ARG", 2: "QP_ERR_UNSUPPORTED_WIDTH", 3: "QP_ERR_PARTITION_MISMATCH",
          4: "QP_ERR_DIM", 5: "QP_ERR_CONFIG_MISMATCH", 6: "QP_ERR_LENGTH", 7: "QP_ERR_ALLOC", 8: "QP_ERR_CUDA",
          9: "QP_ERR_NCCL", 10: "QP_ERR_UNSUPPORTED"}
SCHEMES = {"nuq": 0, "unif": 1, "vq": 2, "tcq": 3, "half_tcq": 4}
DTYPES = {"f16": 0, "bf16": 1, "f32": 2}
QP_X_PREROTATED = 1
QP_NO_PDL = 2
QP_DETERMINISTIC = 4
QP_Y_ACCUMULATE = 8
QP_FUSE_RHT = 16
QP_INDEPENDENT = 32

# every symbol include/qpalette.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "qp_set_allocator", "qp_codebook_load", "qp_codebook_free", "qp_rht_create", "qp_rht_free", "qp_rht_apply",
    "qp_layer_from_codes", "qp_quantize_offline", "qp_quantize_offline_gpu", "qp_layer_get_codes", "qp_layer_get_scales", "qp_linear_fwd",
    "qp_fuse", "qp_group_free", "qp_fused_linear", "qp_dequantize", "qp_layer_shard", "qp_nccl_unique_id",
    "qp_nccl_comm_create", "qp_nccl_comm_destroy", "qp_linear_fwd_sharded", "qp_layer_info", "qp_launch_count",
    "qp_layer_free", "qp_last_error", "qp_version", "qp_shard_range", "qp_optimal_bits", "qp_plan_msq",
    "qp_linear_fwd_sharded_p2p", "qp_ipc_handle", "qp_ipc_open", "qp_ipc_close",
    "qp_codebook_set_scale", "qp_gather_permute", "qp_multi_create", "qp_multi_fwd", "qp_multi_info", "qp_multi_free",
    "qp_multi_fwd_sharded", "qp_multi_fwd_sharded_p2p", "qp_layer_shard_k", "qp_linear_fwd_ksharded",
]


class QPError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2509_20214_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i, sz, u64 = C.c_void_p, C.c_int, C.c_size_t, C.c_uint64
        sig = {
            "qp_codebook_load": [i, i, i, vp, sz, C.POINTER(vp)],
            "qp_codebook_free": [vp],
            "qp_codebook_set_scale": [vp, C.c_double],
            "qp_multi_create": [C.POINTER(vp), i, C.POINTER(vp)],
            "qp_multi_fwd": [vp, C.POINTER(vp), i, i, C.POINTER(vp), i, C.c_uint, vp],
            "qp_multi_info": [vp, C.POINTER(i), C.POINTER(i), C.POINTER(i)],
            "qp_multi_fwd_sharded": [vp, C.POINTER(vp), i, i, C.POINTER(vp), i, vp, C.c_uint, vp],
            "qp_multi_fwd_sharded_p2p": [vp, C.POINTER(vp), i, i, vp, vp, i, i, i, C.c_uint, vp],
            "qp_multi_free": [vp],
            "qp_rht_create": [u64, i, i, C.POINTER(vp)],
            "qp_rht_free": [vp],
            "qp_rht_apply": [vp, vp, i, i, vp, vp],
            "qp_layer_from_codes": [vp, sz, vp, i, i, i, i, vp, vp, C.POINTER(vp)],
            "qp_quantize_offline": [vp, i, i, i, i, vp, vp, i, C.POINTER(vp)],
            "qp_quantize_offline_gpu": [vp, i, i, i, i, vp, vp, i, C.POINTER(vp)],
            "qp_layer_get_codes": [vp, vp, sz],
            "qp_layer_get_scales": [vp, vp],
            "qp_linear_fwd": [vp, vp, i, i, vp, i, C.c_uint, vp],
            "qp_fuse": [C.POINTER(vp), i, C.POINTER(vp)],
            "qp_group_free": [vp],
            "qp_fused_linear": [vp, vp, i, i, C.POINTER(vp), i, C.c_uint, vp],
            "qp_dequantize": [vp, vp, vp],
            "qp_layer_shard": [vp, i, i, C.POINTER(vp)],
            "qp_layer_shard_k": [vp, i, i, C.POINTER(vp)],
            "qp_linear_fwd_ksharded": [vp, vp, i, i, vp, i, vp, C.c_uint, vp],
            "qp_shard_range": [i, i, i, i, i, i, C.POINTER(i), C.POINTER(i), C.POINTER(sz), C.POINTER(sz)],
            "qp_set_allocator": [vp, vp, vp],
            "qp_linear_fwd_sharded_p2p": [vp, vp, i, i, vp, vp, i, i, i, C.c_uint, vp],
            "qp_ipc_handle": [vp, vp],
            "qp_gather_permute": [vp, vp, i, i, i, i, vp],
            "qp_ipc_open": [vp, C.POINTER(vp)],
            "qp_ipc_close": [vp],
            "qp_optimal_bits": [C.POINTER(C.c_double), C.POINTER(C.c_double), i, C.c_double, C.c_double,
                                C.POINTER(C.c_double)],
            "qp_plan_msq": [i, C.POINTER(C.c_double), i, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_double, i,
                            C.POINTER(i), C.POINTER(i), C.POINTER(C.c_double), C.POINTER(C.c_double)],
            "qp_nccl_unique_id": [vp],
            "qp_nccl_comm_create": [vp, i, i, C.POINTER(vp)],
            "qp_nccl_comm_destroy": [vp],
            "qp_linear_fwd_sharded": [vp, vp, i, i, vp, i, vp, C.c_uint, vp],
            "qp_layer_info": [vp, C.POINTER(sz), C.POINTER(C.c_double), C.POINTER(i), C.POINTER(i)],
            "qp_layer_free": [vp],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = None if name.endswith("_free") and name != "qp_nccl_comm_destroy" else C.c_int
        L.qp_last_error.restype = C.c_char_p
        L.qp_version.restype = C.c_char_p
        L.qp_launch_count.restype = C.c_uint64
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != QP_OK:
        raise QPError(status, lib().qp_last_error().decode())


def launch_count() -> int:
    return int(lib().qp_launch_count())


def _ptr(t) -> int:
    """Device (torch) or host (numpy) buffer -> address."""
    if isinstance(t, np.ndarray):
        assert t.flags["C_CONTIGUOUS"]
        return t.ctypes.data
    assert t.is_contiguous(), "tensors passed to the C ABI must be contiguous"
    return t.data_ptr()


def _stream(stream) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dtype_code(t) -> int:
    import torch
    return {torch.float16: 0, torch.bfloat16: 1, torch.float32: 2}[t.dtype]


def gather_permute(src, dst, world: int, batch: int, m: int, stream=None) -> None:
    """qp_gather_permute: [world][batch][m] -> [batch][world * m] (device tensors)."""
    check(lib().qp_gather_permute(_ptr(src), _ptr(dst), world, batch, m, src.element_size(), _stream(stream)))


def shard_range(d_out: int, d_in: int, scheme: str, bits_x4: int, rank: int, world: int):
    """(row0, rows, byte0, nbytes) of rank's row shard (qp_shard_range; host-only, no GPU)."""
    r0, n, b0, nb = C.c_int(), C.c_int(), C.c_size_t(), C.c_size_t()
    check(lib().qp_shard_range(d_out, d_in, SCHEMES[scheme], bits_x4, rank, world, C.byref(r0), C.byref(n),
                               C.byref(b0), C.byref(nb)))
    return r0.value, n.value, b0.value, nb.value


class Codebook:
    """qp_codebook_load: frozen fp16 table (host) -> device decode table."""

    def __init__(self, scheme: str, bits_x4: int, table_fp16: np.ndarray, L: int = 16, alpha: float | None = None):
        t = np.ascontiguousarray(table_fp16, dtype="<f2")
        h = C.c_void_p()
        check(lib().qp_codebook_load(SCHEMES[scheme], bits_x4, L, t.ctypes.data, t.nbytes, C.byref(h)))
        self.h, self.scheme, self.bits_x4, self.L = h, scheme, bits_x4, L
        self.alpha = 1.0
        if alpha is not None:
            self.set_scale(alpha)

    def set_scale(self, alpha: float) -> None:
        """qp_codebook_set_scale: the offline quantizer's reconstruction scale (reading R22)."""
        check(lib().qp_codebook_set_scale(self.h, float(alpha)))
        self.alpha = float(alpha)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.qp_codebook_free(self.h)
            self.h = None


class Rht:
    """qp_rht_create / qp_rht_apply."""

    def __init__(self, seed: int, d_in: int, block: int = 0):
        h = C.c_void_p()
        check(lib().qp_rht_create(seed, d_in, block, C.byref(h)))
        self.h, self.seed, self.d_in = h, seed, d_in

    def apply(self, x, batch: int, out, stream=None) -> None:
        check(lib().qp_rht_apply(self.h, _ptr(x), _dtype_code(x), batch, _ptr(out), _stream(stream)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.qp_rht_free(self.h)
            self.h = None


class Layer:
    """A quantized linear layer (qp_layer)."""

    def __init__(self, handle, codebook: Codebook, rht: Rht):
        self.h = handle
        self._keep = (codebook, rht)
        cb, bpw, do, di = C.c_size_t(), C.c_double(), C.c_int(), C.c_int()
        check(lib().qp_layer_info(self.h, C.byref(cb), C.byref(bpw), C.byref(do), C.byref(di)))
        self.code_bytes, self.bits_per_weight, self.d_out, self.d_in = cb.value, bpw.value, do.value, di.value

    @classmethod
    def from_codes(cls, codes: np.ndarray, scales: np.ndarray, d_out: int, d_in: int, scheme: str, bits_x4: int,
                   codebook: Codebook, rht: Rht) -> "Layer":
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        scales = np.ascontiguousarray(scales, dtype=np.float32)
        h = C.c_void_p()
        check(lib().qp_layer_from_codes(codes.ctypes.data, codes.nbytes, scales.ctypes.data, d_out, d_in,
                                        SCHEMES[scheme], bits_x4, codebook.h, rht.h, C.byref(h)))
        return cls(h, codebook, rht)

    @classmethod
    def quantize_offline(cls, W: np.ndarray, scheme: str, bits_x4: int, codebook: Codebook, rht: Rht,
                         n_threads: int = 0, gpu: bool = False) -> "Layer":
        """gpu=True: the TCQ trellis search runs on the GPU (qp_quantize_offline_gpu)."""
        W = np.ascontiguousarray(W, dtype=np.float32)
        h = C.c_void_p()
        fn = lib().qp_quantize_offline_gpu if gpu else lib().qp_quantize_offline
        check(fn(W.ctypes.data, W.shape[0], W.shape[1], SCHEMES[scheme], bits_x4, codebook.h, rht.h, n_threads,
                 C.byref(h)))
        return cls(h, codebook, rht)

    def codes(self) -> np.ndarray:
        out = np.empty(self.code_bytes, dtype=np.uint8)
        check(lib().qp_layer_get_codes(self.h, out.ctypes.data, out.nbytes))
        return out

    def scales(self) -> np.ndarray:
        out = np.empty(self.d_out, dtype=np.float32)
        check(lib().qp_layer_get_scales(self.h, out.ctypes.data))
        return out

    def forward(self, x, batch: int, y, flags: int = 0, stream=None) -> None:
        """qp_linear_fwd: y[batch][d_out] = diag(s) W_hat R x."""
        check(lib().qp_linear_fwd(self.h, _ptr(x), _dtype_code(x), batch, _ptr(y), _dtype_code(y), flags,
                                  _stream(stream)))

    def dequantize(self, out, stream=None) -> None:
        check(lib().qp_dequantize(self.h, _ptr(out), _stream(stream)))

    def shard(self, rank: int, world: int) -> "Layer":
        h = C.c_void_p()
        check(lib().qp_layer_shard(self.h, rank, world, C.byref(h)))
        return Layer(h, *self._keep)

    def shard_k(self, rank: int, world: int) -> "Layer":
        """qp_layer_shard_k: this rank's input columns (row-parallel layer)."""
        h = C.c_void_p()
        check(lib().qp_layer_shard_k(self.h, rank, world, C.byref(h)))
        return Layer(h, *self._keep)

    def forward_ksharded(self, x_local, batch: int, y, comm, flags: int = 0, stream=None) -> None:
        """qp_linear_fwd_ksharded: partial GEMV on this rank's columns + ncclAllReduce(sum)."""
        check(lib().qp_linear_fwd_ksharded(self.h, _ptr(x_local), _dtype_code(x_local), batch, _ptr(y),
                                           _dtype_code(y), comm.h, flags, _stream(stream)))

    def forward_sharded(self, x, batch: int, y_full, comm, flags: int = 0, stream=None) -> None:
        check(lib().qp_linear_fwd_sharded(self.h, _ptr(x), _dtype_code(x), batch, _ptr(y_full), _dtype_code(y_full),
                                          comm.h, flags, _stream(stream)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.qp_layer_free(self.h)
            self.h = None


class Group:
    """qp_fuse / qp_fused_linear (fused QKV or up-gate)."""

    def __init__(self, members: list[Layer]):
        arr = (C.c_void_p * len(members))(*[m.h for m in members])
        h = C.c_void_p()
        check(lib().qp_fuse(arr, len(members), C.byref(h)))
        self.h = h
        self.d_outs = [m.d_out for m in members]
        self._keep = members[0]._keep

    def forward(self, x, batch: int, ys: list, flags: int = 0, stream=None) -> None:
        arr = (C.c_void_p * len(ys))(*[_ptr(y) for y in ys])
        check(lib().qp_fused_linear(self.h, _ptr(x), _dtype_code(x), batch, arr, _dtype_code(ys[0]), flags,
                                    _stream(stream)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.qp_group_free(self.h)
            self.h = None


class Multi:
    """qp_multi_*: the persistent multi-layer engine -- one launch runs the rotations and fused
    dequant-GEMVs of a list of independent layers that share a decode table."""

    def __init__(self, layers: list[Layer]):
        arr = (C.c_void_p * len(layers))(*[l.h for l in layers])
        h = C.c_void_p()
        check(lib().qp_multi_create(arr, len(layers), C.byref(h)))
        self.h = h
        self.layers = list(layers)
        n, nl, ne = C.c_int(), C.c_int(), C.c_int()
        check(lib().qp_multi_info(self.h, C.byref(n), C.byref(nl), C.byref(ne)))
        self.n_layers, self.n_launches, self.n_engine_launches = n.value, nl.value, ne.value

    def forward(self, xs: list, batch: int, ys: list, flags: int = 0, stream=None) -> None:
        """y_i = diag(s_i) W_hat_i R_i x_i for every layer i (qp_multi_fwd)."""
        assert len(xs) == len(ys) == len(self.layers)
        xa = (C.c_void_p * len(xs))(*[_ptr(x) for x in xs])
        ya = (C.c_void_p * len(ys))(*[_ptr(y) for y in ys])
        check(lib().qp_multi_fwd(self.h, xa, _dtype_code(xs[0]), batch, ya, _dtype_code(ys[0]), flags,
                                 _stream(stream)))

    def forward_sharded(self, xs: list, batch: int, ys_full: list, comm, flags: int = 0, stream=None) -> None:
        """qp_multi_fwd_sharded: the layers are shards; ys_full[i] receives all ranks' rows."""
        xa = (C.c_void_p * len(xs))(*[_ptr(x) for x in xs])
        ya = (C.c_void_p * len(ys_full))(*[_ptr(y) for y in ys_full])
        check(lib().qp_multi_fwd_sharded(self.h, xa, _dtype_code(xs[0]), batch, ya, _dtype_code(ys_full[0]), comm.h,
                                         flags, _stream(stream)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.qp_multi_free(self.h)
            self.h = None


class NcclComm:
    """NCCL communicator of the sharded path; the 128-byte unique id is exchanged by the caller."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_char * 128)()
        check(lib().qp_nccl_unique_id(buf))
        return bytes(buf)

    def __init__(self, uid: bytes, world: int, rank: int):
        buf = (C.c_char * 128).from_buffer_copy(uid)
        h = C.c_void_p()
        check(lib().qp_nccl_comm_create(buf, world, rank, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            check(lib().qp_nccl_comm_destroy(self.h))
            self.h = None


def optimal_bits(a, n, M: float, eta: float) -> np.ndarray:
    """qp_optimal_bits (host-only): Theorem 1 allocation b_l* for sensitivities a, sizes n."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    n = np.ascontiguousarray(n, dtype=np.float64)
    out = np.empty_like(a)
    dp = C.POINTER(C.c_double)
    check(lib().qp_optimal_bits(a.ctypes.data_as(dp), n.ctypes.data_as(dp), len(a), float(M), float(eta),
                                out.ctypes.data_as(dp)))
    return out


def plan_msq(a, err, cost, budget: float, fusion: bool = True):
    """qp_plan_msq (host-only): a [B][7], err [nq], cost [12][nq] -> (loss, cost, group [B][7], quant [B][7])."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    err = np.ascontiguousarray(err, dtype=np.float64)
    cost = np.ascontiguousarray(cost, dtype=np.float64)
    B, nq = a.shape[0], err.shape[0]
    g = np.full((B, 7), -1, dtype=np.int32)
    q = np.full((B, 7), -1, dtype=np.int32)
    lo, co = C.c_double(), C.c_double()
    dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int)
    check(lib().qp_plan_msq(B, a.ctypes.data_as(dp), nq, err.ctypes.data_as(dp), cost.ctypes.data_as(dp), float(budget),
                            1 if fusion else 0, g.ctypes.data_as(ip), q.ctypes.data_as(ip), C.byref(lo), C.byref(co)))
    return lo.value, co.value, g, q


_ALLOC_CB = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
_FREE_CB = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)
_allocator_refs = None


def use_torch_allocator(enable: bool = True) -> None:
    """Route the library's device allocations (codes, scales, tables, workspaces) through
    PyTorch's caching allocator (qp_set_allocator), so one memory pool serves both. Affects
    objects created afterwards; free them before disabling."""
    global _allocator_refs
    import torch
    if not enable:
        check(lib().qp_set_allocator(None, None, None))
        _allocator_refs = None
        return

    def alloc(n, ctx):
        try:
            return int(torch.cuda.caching_allocator_alloc(max(int(n), 1)))
        except Exception:           # out of memory -> NULL -> QP_ERR_ALLOC
            return None

    def free(ptr, ctx):
        if ptr:
            torch.cuda.caching_allocator_delete(int(ptr))

    _allocator_refs = (_ALLOC_CB(alloc), _FREE_CB(free))     # keep the thunks alive
    check(lib().qp_set_allocator(C.cast(_allocator_refs[0], C.c_void_p), C.cast(_allocator_refs[1], C.c_void_p), None))


class PeerGather:
    """Fused all-gather destination for row-sharded layers (qp_linear_fwd_sharded_p2p): every
    rank allocates y_full [batch][world * m] and a flag array, exchanges CUDA IPC handles through
    torch.distributed (`group`, any backend) and maps its peers' buffers. world == 1 needs no
    process group."""

    def __init__(self, world: int, rank: int, m: int, batch: int, dtype=None, group=None):
        import torch
        dtype = dtype or torch.float32
        self.world, self.rank, self.m, self.batch = world, rank, m, batch
        self.y = torch.zeros(batch, world * m, dtype=dtype, device="cuda")
        self.flags = torch.zeros(2 * world + 1, dtype=torch.int32, device="cuda")   # delivered | consumed | entered
        self._opened = []
        if world == 1:
            ys, fs = [self.y.data_ptr()], [self.flags.data_ptr()]
        else:
            import torch.distributed as dist
            hy, hf = (C.c_char * 72)(), (C.c_char * 72)()
            check(lib().qp_ipc_handle(C.c_void_p(self.y.data_ptr()), hy))
            check(lib().qp_ipc_handle(C.c_void_p(self.flags.data_ptr()), hf))
            allh = [None] * world
            dist.all_gather_object(allh, (bytes(hy), bytes(hf)), group=group)
            ys, fs = [], []
            for k, (by, bf) in enumerate(allh):
                if k == rank:
                    ys.append(self.y.data_ptr())
                    fs.append(self.flags.data_ptr())
                    continue
                py, pf = C.c_void_p(), C.c_void_p()
                check(lib().qp_ipc_open(by, C.byref(py)))
                check(lib().qp_ipc_open(bf, C.byref(pf)))
                self._opened += [py.value, pf.value]
                ys.append(py.value)
                fs.append(pf.value)
            torch.cuda.synchronize()
            dist.barrier(group=group)
        self._ys = (C.c_void_p * world)(*ys)
        self._fs = (C.c_void_p * world)(*fs)

    def forward(self, shard: "Layer", x, flags: int = 0, stream=None) -> None:
        check(lib().qp_linear_fwd_sharded_p2p(shard.h, _ptr(x), _dtype_code(x), self.batch, self._ys, self._fs,
                                              self.rank, self.world, _dtype_code(self.y), flags, _stream(stream)))

    def close(self):
        for p in self._opened:
            lib().qp_ipc_close(C.c_void_p(p))
        self._opened = []


class MultiPeerGather:
    """Fused all-gather destinations of a qp_multi over row shards (qp_multi_fwd_sharded_p2p): one
    device buffer holds every layer's y_full [batch][world * m_i] (self.ys[i] are views), plus the
    flag array; the two CUDA IPC handles are exchanged through torch.distributed (`group`, any
    backend) and the peers' buffers mapped. world == 1 needs no process group."""

    def __init__(self, world: int, rank: int, ms: list, batch: int, dtype=None, group=None):
        import torch
        dtype = dtype or torch.float32
        self.world, self.rank, self.ms, self.batch = world, rank, list(ms), batch
        eb = torch.empty(0, dtype=dtype).element_size()
        # 256-byte aligned slices of one allocation
        self._offs, off = [], 0
        for m in self.ms:
            self._offs.append(off)
            off += (batch * world * m * eb + 255) // 256 * 256
        self.buf = torch.zeros(off, dtype=torch.uint8, device="cuda")
        self.ys = [self.buf[o:o + batch * world * m * eb].view(dtype).view(batch, world * m)
                   for o, m in zip(self._offs, self.ms)]
        self.flags = torch.zeros(2 * world + 1, dtype=torch.int32, device="cuda")
        self._opened = []
        if world == 1:
            bases, fs = [self.buf.data_ptr()], [self.flags.data_ptr()]
        else:
            import torch.distributed as dist
            hb, hf = (C.c_char * 72)(), (C.c_char * 72)()
            check(lib().qp_ipc_handle(C.c_void_p(self.buf.data_ptr()), hb))
            check(lib().qp_ipc_handle(C.c_void_p(self.flags.data_ptr()), hf))
            allh = [None] * world
            dist.all_gather_object(allh, (bytes(hb), bytes(hf)), group=group)
            bases, fs = [], []
            for k, (bb, bf) in enumerate(allh):
                if k == rank:
                    bases.append(self.buf.data_ptr())
                    fs.append(self.flags.data_ptr())
                    continue
                pb, pf = C.c_void_p(), C.c_void_p()
                check(lib().qp_ipc_open(bb, C.byref(pb)))
                check(lib().qp_ipc_open(bf, C.byref(pf)))
                self._opened += [pb.value, pf.value]
                bases.append(pb.value)
                fs.append(pf.value)
            torch.cuda.synchronize()
            dist.barrier(group=group)
        n = len(self.ms)
        self._ys = (C.c_void_p * (n * world))(*[bases[k] + self._offs[i] for i in range(n) for k in range(world)])
        self._fs = (C.c_void_p * world)(*fs)

    def forward(self, multi: "Multi", xs: list, flags: int = 0, stream=None) -> None:
        assert len(xs) == len(self.ms) == multi.n_layers
        xa = (C.c_void_p * len(xs))(*[_ptr(x) for x in xs])
        check(lib().qp_multi_fwd_sharded_p2p(multi.h, xa, _dtype_code(xs[0]), self.batch, self._ys, self._fs,
                                             self.rank, self.world, _dtype_code(self.ys[0]), flags,
                                             _stream(stream)))

    def close(self):
        for p in self._opened:
            lib().qp_ipc_close(C.c_void_p(p))
        self._opened = []
