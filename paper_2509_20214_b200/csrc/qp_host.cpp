// Host side of the C ABI (include/qpalette.h): validation, object lifetime, codebook
// expansion into device decode tables, layer / group / shard objects, NCCL glue and the
// data-free offline quantizer (weight RHT, scales, RTN, rotate-half tail-biting Viterbi).
//
// Paper passages: P:345-349 (rotation + scales), P:975 (data-free procedure),
// P:977-1065 (quantizer definitions), P:359-360 (bit-packing, table-lookup merging),
// P:456-460 (layer fusion). Layout: LAYOUT.md. Readings R1-R20: DESIGN.md.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <limits>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/qpalette.h"
#include "qp_internal.h"

using namespace qp;

// ---------------------------------------------------------------------------------------
// errors, allocation, launch accounting
// ---------------------------------------------------------------------------------------
namespace {
thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};
void* (*g_alloc)(size_t, void*) = nullptr;
void (*g_free)(void*, void*) = nullptr;
void* g_alloc_ctx = nullptr;

qp_status fail(qp_status s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}
qp_status cuda_fail(cudaError_t e, const char* what) {
  return fail(QP_ERR_CUDA, "%s: %s (%s). Remedy: run on an sm_100 (B200) GPU with a matching driver; check inputs "
              "are device pointers.", what, cudaGetErrorName(e), cudaGetErrorString(e));
}
#define CUDA_TRY(expr, what)                  \
  do {                                        \
    cudaError_t e_ = (expr);                  \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

void* dev_alloc(size_t n) {
  if (n == 0) n = 16;
  if (g_alloc) return g_alloc(n, g_alloc_ctx);
  void* p = nullptr;
  return cudaMalloc(&p, n) == cudaSuccess ? p : nullptr;
}
void dev_free(void* p) {
  if (!p) return;
  if (g_free) g_free(p, g_alloc_ctx);
  else cudaFree(p);
}

// QP_NO_PDL=1 in the environment disables programmatic dependent launch (profilers such as
// ncu cannot replay PDL edges inside captured CUDA graphs).
bool pdl_disabled_by_env() {
  static const bool off = [] {
    const char* e = getenv("QP_NO_PDL");
    return e && e[0] == '1';
  }();
  return off;
}

bool f16_inorder_by_env() {   // QP_F16_INORDER=1: fp16 y through the in-order epilogue (experiments)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("QP_F16_INORDER");
    v = (e && atoi(e) != 0) ? 1 : 0;
  }
  return v == 1;
}

bool fused_rht_by_env() {   // QP_FUSED_RHT=1: QP_FUSE_RHT on every forward (experiments)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("QP_FUSED_RHT");
    v = (e && atoi(e) != 0) ? 1 : 0;
  }
  return v == 1;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

uint16_t f32_to_f16_bits(float f) {
  __half h = __float2half_rn(f);
  uint16_t b;
  std::memcpy(&b, &h, 2);
  return b;
}
float f16_bits_to_f32(uint16_t b) {
  __half h;
  std::memcpy(&h, &b, 2);
  return __half2float(h);
}

// splitmix64 counter generator (reading R8): i-th output for seed.
uint64_t splitmix64(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int tlut_bits_for_x4(int bits_x4) {  // 9 for b <= 4, 10 for 4.5, 11 for 5.0
  if (bits_x4 <= 16) return 9;
  if (bits_x4 <= 18) return 10;
  return 11;
}

bool width_ok(qp_scheme s, int x4) {
  switch (s) {
    case QP_TCQ: return x4 >= 6 && x4 <= 20 && x4 % 2 == 0;
    case QP_HALF_TCQ: return x4 >= 7 && x4 <= 19 && x4 % 2 == 1;
    case QP_VQ: return x4 >= 6 && x4 <= 24 && x4 % 2 == 0;
    case QP_NUQ:
    case QP_UNIF: return x4 >= 8 && x4 <= 32 && x4 % 4 == 0;
  }
  return false;
}

// bits per 2-weight step for k-tiles in the low / high half of d_in
void step_bits(qp_scheme s, int x4, int* c_lo, int* c_hi) {
  if (s == QP_HALF_TCQ) {
    *c_lo = (x4 - 1) / 2;
    *c_hi = *c_lo + 1;
  } else {
    *c_lo = *c_hi = x4 / 2;
  }
}
}  // namespace

namespace qp {
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace qp

// ---------------------------------------------------------------------------------------
// objects
// ---------------------------------------------------------------------------------------
struct qp_codebook {
  qp_scheme scheme;
  int bits_x4;
  int L;         // TCQ window bits
  int tb;        // tlut bits (TCQ) or scalar code bits (NUQ/UNIF)
  int mode;      // qp::DecMode
  int reps;
  double alpha = 1.0;           // reconstruction scale of the offline quantizer (reading R22)
  std::vector<uint16_t> host;   // the loaded fp16 table
  uint32_t* d_table = nullptr;  // compact device table (half2 words)
  int table_words = 0;
};

struct qp_rht {
  uint64_t seed;
  int d_in, block;
  std::vector<uint32_t> sign_bits;  // bit i = 1 -> d_i = -1
  uint32_t* d_signs = nullptr;
};

struct qp_layer {
  int d_out = 0, d_in = 0;
  qp_scheme scheme;
  int bits_x4 = 0, c_lo = 0, c_hi = 0;
  size_t code_bytes = 0;
  uint8_t* d_codes = nullptr;
  float* d_scales = nullptr;
  const qp_codebook* cb = nullptr;
  const qp_rht* rht = nullptr;
  KernelKey key{};
  GemvLauncher launcher = nullptr;
  int grid = 0;
  float* d_ws = nullptr;
  int* d_counters = nullptr;
  __half* d_xrot = nullptr;   // [8][d_in] scratch for R x
  float* d_yws = nullptr;     // [8][d_out] fp32 accumulation workspace for fp16 y
  void* d_gather = nullptr;   // sharded path scratch
  size_t gather_bytes = 0;
  qp_rht* owned_rht = nullptr;  // k-shards: the column slice of the parent's rotation (freed with the layer)
};

struct qp_group {
  qp_layer* cat = nullptr;          // concatenated rows
  std::vector<int> d_outs;
};

namespace {

qp_status make_kernel_key(const qp_codebook* cb, qp_scheme scheme, int c_lo, int c_hi, KernelKey* k) {
  if (scheme == QP_TCQ || scheme == QP_HALF_TCQ) {
    *k = KernelKey{cb->mode, c_lo, c_hi, cb->L, cb->tb, cb->reps};
  } else if (scheme == QP_VQ) {
    *k = KernelKey{DEC_LUT2, c_lo, c_lo, 0, 0, cb->reps};
  } else {
    if (cb->mode == DEC_LUT2) *k = KernelKey{DEC_LUT2, c_lo, c_lo, 0, 0, cb->reps};
    else *k = KernelKey{DEC_SCALAR, c_lo, c_lo, 0, cb->tb, cb->reps};
  }
  // the kernels expand exactly this many compact-table words (TableBuild, no bounds checks)
  const int entries = k->mode == DEC_TCQ_PRESIGNED ? (2 << k->tb) : k->mode == DEC_LUT2 ? (1 << k->c_lo) : (1 << k->tb);
  if (cb->table_words != entries)
    return fail(QP_ERR_CONFIG_MISMATCH, "codebook table has %d words, the decoder expects %d", cb->table_words, entries);
  return QP_OK;
}

qp_status check_codebook(const qp_codebook* cb, qp_scheme scheme, int bits_x4) {
  if (!cb) return fail(QP_ERR_INVALID_ARG, "codebook is NULL. Remedy: load one with qp_codebook_load.");
  const bool tcq_family = scheme == QP_TCQ || scheme == QP_HALF_TCQ;
  const bool cb_tcq = cb->scheme == QP_TCQ || cb->scheme == QP_HALF_TCQ;
  if (tcq_family != cb_tcq || (!tcq_family && cb->scheme != scheme))
    return fail(QP_ERR_CONFIG_MISMATCH, "codebook scheme %d does not serve layer scheme %d. Remedy: load the codebook "
                "of the layer's quantizer.", (int)cb->scheme, (int)scheme);
  if (tcq_family) {
    const int need_tb = tlut_bits_for_x4(scheme == QP_HALF_TCQ ? bits_x4 + 1 : bits_x4);
    if (cb->tb != need_tb)
      return fail(QP_ERR_CONFIG_MISMATCH, "TCQ width %.2f needs tlut_bits %d (P:1036), codebook has %d. Remedy: load "
                  "the matching tlut.", bits_x4 / 4.0, need_tb, cb->tb);
  } else if (scheme == QP_VQ) {
    if (cb->bits_x4 != bits_x4)
      return fail(QP_ERR_CONFIG_MISMATCH, "VQ codebook is %.1f bits, layer %.1f. Remedy: load the matching LUT.",
                  cb->bits_x4 / 4.0, bits_x4 / 4.0);
  } else if (cb->bits_x4 != bits_x4) {
    return fail(QP_ERR_CONFIG_MISMATCH, "scalar codebook is %d bits, layer %d. Remedy: load the matching LUT.",
                cb->bits_x4 / 4, bits_x4 / 4);
  }
  return QP_OK;
}

qp_status check_shape(qp_scheme scheme, int bits_x4, int d_out, int d_in) {
  if (!width_ok(scheme, bits_x4))
    return fail(QP_ERR_UNSUPPORTED_WIDTH, "scheme %d does not support %.2f bits (Table 1, P:192-211). Remedy: pick a "
                "width from include/qpalette.h.", (int)scheme, bits_x4 / 4.0);
  if (d_out <= 0 || d_in <= 0) return fail(QP_ERR_DIM, "d_out and d_in must be positive");
  if (d_out % kTileRows || d_in % kTileCols)
    return fail(QP_ERR_PARTITION_MISMATCH, "d_out=%d must be a multiple of 32 and d_in=%d of 256 (LAYOUT.md tiles). "
                "Remedy: pad the layer.", d_out, d_in);
  if (scheme == QP_HALF_TCQ && (d_in / 2) % kTileCols)
    return fail(QP_ERR_PARTITION_MISMATCH, "half-TCQ needs (d_in/2) %% 256 == 0 (P:297); d_in=%d", d_in);
  return QP_OK;
}

size_t layout_bytes(qp_scheme scheme, int bits_x4, int d_out, int d_in) {
  int c_lo, c_hi;
  step_bits(scheme, bits_x4, &c_lo, &c_hi);
  const size_t RT = d_out / kTileRows, KT = d_in / kTileCols, KH = KT / 2;
  return RT * (KH * 512 * (size_t)c_lo + (KT - KH) * 512 * (size_t)c_hi);
}

// Allocate the device side of a layer whose codes/scales are given on the device or host.
qp_status layer_init(qp_layer* l, int d_out, int d_in, qp_scheme scheme, int bits_x4, const qp_codebook* cb,
                     const qp_rht* r) {
  l->d_out = d_out;
  l->d_in = d_in;
  l->scheme = scheme;
  l->bits_x4 = bits_x4;
  step_bits(scheme, bits_x4, &l->c_lo, &l->c_hi);
  l->code_bytes = layout_bytes(scheme, bits_x4, d_out, d_in);
  l->cb = cb;
  l->rht = r;
  if (qp_status st = make_kernel_key(cb, scheme, l->c_lo, l->c_hi, &l->key); st != QP_OK) return st;
  l->launcher = find_gemv(l->key);
  if (!l->launcher)
    return fail(QP_ERR_UNSUPPORTED, "no compiled kernel variant for mode=%d c=%d/%d L=%d tb=%d reps=%d. Remedy: add it "
                "to the qp_inst_*.cu instantiation lists.", l->key.mode, l->key.c_lo, l->key.c_hi, l->key.L,
                l->key.tb, l->key.reps);
  const long long ntiles = (long long)(d_out / kTileRows) * (d_in / kTileCols);
  l->grid = (int)std::min<long long>(num_sms(), ntiles);
  if ((unsigned long long)ntiles * (unsigned long long)(l->grid + 1) >= (1ull << 32))
    return fail(QP_ERR_DIM, "layer of %lld tiles is too large for 32-bit tile indexing", ntiles);
  l->d_codes = static_cast<uint8_t*>(dev_alloc(l->code_bytes));
  l->d_scales = static_cast<float*>(dev_alloc((size_t)d_out * 4));
  l->d_ws = static_cast<float*>(dev_alloc((size_t)l->grid * 256 * 4));
  l->d_counters = static_cast<int*>(dev_alloc((size_t)(d_out / kTileRows + 2) * 4));   // + grid barrier [2]
  l->d_xrot = static_cast<__half*>(dev_alloc((size_t)8 * d_in * 2));
  l->d_yws = static_cast<float*>(dev_alloc((size_t)8 * d_out * 4));
  if (!l->d_codes || !l->d_scales || !l->d_ws || !l->d_counters || !l->d_xrot || !l->d_yws)
    return fail(QP_ERR_ALLOC, "device allocation of %zu code bytes failed", l->code_bytes);
  CUDA_TRY(cudaMemset(l->d_counters, 0, (size_t)(d_out / kTileRows + 2) * 4), "cudaMemset(counters)");
  // the memset runs on the legacy default stream, which PyTorch's (non-blocking) streams do not
  // order against: complete it before the layer is handed out
  CUDA_TRY(cudaStreamSynchronize(0), "cudaStreamSynchronize(layer init)");
  return QP_OK;
}

void layer_release(qp_layer* l) {
  if (!l) return;
  dev_free(l->d_codes);
  dev_free(l->d_scales);
  dev_free(l->d_ws);
  dev_free(l->d_counters);
  dev_free(l->d_xrot);
  dev_free(l->d_yws);
  dev_free(l->d_gather);
  if (l->owned_rht) {
    dev_free(l->owned_rht->d_signs);
    delete l->owned_rht;
    l->owned_rht = nullptr;
  }
}

qp_status run_rht(const qp_rht* r, const void* x, qp_dtype xt, int batch, __half* out, bool pdl, cudaStream_t s,
                  int n_zero = 0, void* const* zero_ptr = nullptr, const long long* zero_n = nullptr) {
  RhtParams p{};
  p.n_zero = n_zero;
  for (int i = 0; i < n_zero; ++i) {
    p.zero_ptr[i] = static_cast<float*>(zero_ptr[i]);
    p.zero_n[i] = zero_n[i];
  }
  p.x = x;
  p.x_dtype = (int)xt;
  p.batch = batch;
  p.d_in = r->d_in;
  p.block = r->block;
  p.signs = r->d_signs;
  p.out = out;
  p.scale = (float)(1.0 / std::sqrt((double)r->block));
  cudaError_t e = launch_rht(p, pdl, s);
  if (e != cudaSuccess) return cuda_fail(e, "rht kernel launch");
  return QP_OK;
}

// ceil(2^32 / d) when floor(x / d) == __umulhi(x, m) for every x <= x_max (x * (m*d - 2^32) < 2^32
// suffices since m*d - 2^32 < d), else 0 (the kernel then divides).
uint32_t div_magic(uint64_t d, uint64_t x_max) {
  if (d <= 1 || x_max * d >= (1ull << 32)) return 0;
  return (uint32_t)(((1ull << 32) + d - 1) / d);
}

void set_magics(GemvParams& p, int grid) {
  const uint64_t N = (uint64_t)p.RT * (uint64_t)p.KT;
  p.kt_magic = div_magic((uint64_t)p.KT, N + 8);
  p.grid_magic = div_magic((uint64_t)grid, N * (uint64_t)grid);
}

// CTAs of the zeroing kernel: one per 64 KB of fp32 output, 1..8
int zero_ctas(const long long* zn, int n) {
  long long bytes = 0;
  for (int i = 0; i < n; ++i) bytes += zn[i] * 4;
  return (int)std::max<long long>(1, std::min<long long>(8, (bytes + 65535) / 65536));
}

// side_ctas: CTAs of the preceding rotation / zeroing kernel. Under PDL the GEMV (one CTA per SM,
// the whole register file) cannot share an SM with them, so a GEMV CTA placed there would start
// its prologue only after they exit and finish last; the GEMV leaves those SMs to them instead.
// Fused rotation request for run_gemv: x' = R x computed inside the GEMV kernel (and, for the
// fp32 atomic path, y zeroed there too); run_gemv reports `unsupported` (nothing launched) when
// the layer / batch does not fit the fused plan, and the caller launches the rotation kernel.
struct FusedRot {
  const qp_rht* r;
  const void* x;
  qp_dtype xt;
  bool zero_y;
};

// Fused all-gather destination for run_gemv (qp_linear_fwd_sharded_p2p)
struct PeerOut {
  int world, rank, row0, ld;
  void* const* y;
  unsigned* const* flag;
};
thread_local const PeerOut* g_peer_out = nullptr;   // set around one run_gemv call

qp_status run_gemv(const qp_layer* l, const __half* xr, int batch, int n_out, const int* rt_begin, void* const* ys,
                   const int* ldy, qp_dtype yt, bool pdl, cudaStream_t s, bool y_atomic, int side_ctas = 0,
                   const FusedRot* fr = nullptr, bool* unsupported = nullptr, bool y_accum = false) {
  GemvParams p{};
  p.y_accum = y_accum ? 1 : 0;
  if (y_atomic && yt == QP_F16) {                 // fp16 y via the fp32 workspace (zeroed by the caller)
    p.y_ws = 1;
    for (int i = 0; i < n_out; ++i) p.yws[i] = l->d_yws + (size_t)batch * rt_begin[i] * kTileRows;
  }
  if (g_peer_out) {
    p.n_peers = g_peer_out->world;
    for (int k = 0; k < g_peer_out->world; ++k) {
      p.peer_y[k] = g_peer_out->y[k];
      p.peer_flag[k] = g_peer_out->flag[k];
    }
    p.peer_rank = g_peer_out->rank;
    p.peer_row0 = g_peer_out->row0;
    p.peer_ld = g_peer_out->ld;
    p.peer_counter = l->d_counters + l->d_out / kTileRows;   // (the fused-rotation barrier's slot)
  }
  if (fr) {
    p.x_raw = fr->x;
    p.x_dtype = (int)fr->xt;
    p.rht_block = fr->r->block;
    p.rht_signs = fr->r->d_signs;
    p.rht_scale = (float)(1.0 / std::sqrt((double)fr->r->block));
    p.zero_y = fr->zero_y ? 1 : 0;
    p.bar_count = l->d_counters + l->d_out / kTileRows;
  }
  p.y_atomic = y_atomic ? 1 : 0;
  p.codes = l->d_codes;
  p.scales = l->d_scales;
  p.table = l->cb->d_table;
  p.table_words = l->cb->table_words;
  p.RT = l->d_out / kTileRows;
  p.KT = l->d_in / kTileCols;
  p.d_in = l->d_in;
  p.batch = batch;
  p.x = xr;
  p.n_out = n_out;
  for (int i = 0; i <= n_out; ++i) p.rt_begin[i] = rt_begin[i];
  for (int i = 0; i < n_out; ++i) {
    p.y[i] = ys[i];
    p.ldy[i] = ldy[i];
  }
  p.y_f32 = yt == QP_F32 ? 1 : 0;
  p.ws = l->d_ws;
  p.counters = l->d_counters;
  int grid = l->grid;
  if (pdl && side_ctas > 0 && side_ctas <= kMaxSideCtas) grid = std::max(1, std::min(grid, num_sms() - side_ctas));
  set_magics(p, grid);
  cudaError_t e = l->launcher(p, grid, 0, false, pdl, s);
  if (e == cudaErrorNotSupported && fr && unsupported) {
    *unsupported = true;
    return QP_OK;
  }
  if (e != cudaSuccess) return cuda_fail(e, "fused dequant-GEMV launch");
  count_launch();
  return QP_OK;
}

qp_status check_fwd_args(const void* x, qp_dtype xt, int batch, qp_dtype yt, unsigned flags) {
  if (!x) return fail(QP_ERR_INVALID_ARG, "x is NULL");
  if (batch < 1 || batch > 8)
    return fail(QP_ERR_PARTITION_MISMATCH, "batch=%d outside 1..8 (P:292). Remedy: split the batch.", batch);
  if ((int)xt < 0 || (int)xt > 2 || (yt != QP_F32 && yt != QP_F16))
    return fail(QP_ERR_INVALID_ARG, "dtype: x in {F16,BF16,F32}, y in {F16,F32}");
  if ((flags & QP_X_PREROTATED) && xt != QP_F16)
    return fail(QP_ERR_INVALID_ARG, "QP_X_PREROTATED requires fp16 x (the output dtype of qp_rht_apply)");
  if ((flags & QP_X_PREROTATED) && (reinterpret_cast<uintptr_t>(x) & 31u))
    return fail(QP_ERR_INVALID_ARG, "QP_X_PREROTATED x must be 32-byte aligned (the GEMV reads it with 256-bit "
                "loads). Remedy: pass the start of a device allocation");
  if ((flags & QP_Y_ACCUMULATE) && (yt != QP_F32 || (flags & QP_DETERMINISTIC)))
    return fail(QP_ERR_INVALID_ARG, "QP_Y_ACCUMULATE needs fp32 y and excludes QP_DETERMINISTIC");
  return QP_OK;
}

}  // namespace

namespace qp {
int set_error(int status, const char* msg) { return (int)fail((qp_status)status, "%s", msg); }
}  // namespace qp

// ---------------------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------------------
extern "C" {

const char* qp_last_error(void) { return g_err.c_str(); }
const char* qp_version(void) { return "qpalette-b200 0.1 (sm_100a)"; }
uint64_t qp_launch_count(void) { return g_launches.load(); }

qp_status qp_set_allocator(void* (*alloc)(size_t, void*), void (*free_)(void*, void*), void* ctx) {
  if ((alloc == nullptr) != (free_ == nullptr)) return fail(QP_ERR_INVALID_ARG, "give both alloc and free, or neither");
  g_alloc = alloc;
  g_free = free_;
  g_alloc_ctx = ctx;
  return QP_OK;
}

qp_status qp_codebook_load(qp_scheme scheme, int bits_x4, int L, const void* host_fp16, size_t n_bytes,
                           qp_codebook** out) {
  if (!host_fp16 || !out) return fail(QP_ERR_INVALID_ARG, "NULL argument to qp_codebook_load");
  *out = nullptr;
  if (!width_ok(scheme, bits_x4)) return fail(QP_ERR_UNSUPPORTED_WIDTH, "unsupported width %.2f", bits_x4 / 4.0);
  auto cb = new qp_codebook();
  cb->scheme = scheme;
  cb->bits_x4 = bits_x4;
  cb->L = 0;
  const uint16_t* h = static_cast<const uint16_t*>(host_fp16);
  std::vector<uint32_t> words;
  size_t expect = 0;
  if (scheme == QP_TCQ || scheme == QP_HALF_TCQ) {
    if (L != 16 && L != 12) {
      delete cb;
      return fail(QP_ERR_CONFIG_MISMATCH, "L=%d; supported trellis windows are 16 (P:1043) and 12 (config C1)", L);
    }
    cb->L = L;
    cb->tb = tlut_bits_for_x4(scheme == QP_HALF_TCQ ? bits_x4 + 1 : bits_x4);
    expect = ((size_t)1 << cb->tb) * 4;
    if (n_bytes != expect) {
      delete cb;
      return fail(QP_ERR_LENGTH, "tlut for tlut_bits=%d must be %zu bytes, got %zu", cb->tb, expect, n_bytes);
    }
    const int n = 1 << cb->tb;
    if (cb->tb == 9) {
      // pre-signed key table: key = sign * 2^tb + idx -> (sign ? -t0 : t0, t1)
      cb->mode = DEC_TCQ_PRESIGNED;
      // 32 replicas (bank = lane, conflict-free). 16 replicas would save the shift of the key
      // (one instruction per pair) but measured 5-15% slower on B200 with the 2-way bank
      // conflicts (profiles/r1/ubench_decode_variants.txt)
      cb->reps = 32;
      words.resize(2 * n);
      for (int sgn = 0; sgn < 2; ++sgn)
        for (int i = 0; i < n; ++i) {
          const uint32_t t0 = h[2 * i] ^ (sgn ? 0x8000u : 0u), t1 = h[2 * i + 1];
          words[sgn * n + i] = t0 | (t1 << 16);
        }
    } else {
      cb->mode = DEC_TCQ_UNSIGNED;
      cb->reps = cb->tb == 10 ? 32 : 16;
      words.resize(n);
      for (int i = 0; i < n; ++i) words[i] = (uint32_t)h[2 * i] | ((uint32_t)h[2 * i + 1] << 16);
    }
  } else if (scheme == QP_VQ) {
    const int c = bits_x4 / 2;
    expect = ((size_t)1 << c) * 4;
    if (n_bytes != expect) {
      delete cb;
      return fail(QP_ERR_LENGTH, "VQ-%.1f LUT must be %zu bytes, got %zu", bits_x4 / 4.0, expect, n_bytes);
    }
    cb->mode = DEC_LUT2;
    cb->reps = c <= 10 ? 32 : (c == 11 ? 16 : 8);
    words.resize((size_t)1 << c);
    for (size_t i = 0; i < words.size(); ++i) words[i] = (uint32_t)h[2 * i] | ((uint32_t)h[2 * i + 1] << 16);
  } else {
    const int b = bits_x4 / 4;
    expect = ((size_t)1 << b) * 2;
    if (n_bytes != expect) {
      delete cb;
      return fail(QP_ERR_LENGTH, "scalar LUT of %d bits must be %zu bytes, got %zu", b, expect, n_bytes);
    }
    cb->tb = b;
    if (b <= 4) {
      // table-lookup merging: pair index c_even * 2^b + c_odd
      cb->mode = DEC_LUT2;
      cb->reps = 32;
      const int n = 1 << b;
      words.resize((size_t)n * n);
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) words[i * n + j] = (uint32_t)h[i] | ((uint32_t)h[j] << 16);
    } else {
      cb->mode = DEC_SCALAR;
      cb->reps = 32;
      words.resize((size_t)1 << b);
      for (size_t i = 0; i < words.size(); ++i) words[i] = h[i];
    }
  }
  cb->host.assign(h, h + n_bytes / 2);
  cb->table_words = (int)words.size();
  cb->d_table = static_cast<uint32_t*>(dev_alloc(words.size() * 4));
  if (!cb->d_table) {
    delete cb;
    return fail(QP_ERR_ALLOC, "codebook table allocation failed");
  }
  cudaError_t e = cudaMemcpy(cb->d_table, words.data(), words.size() * 4, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    dev_free(cb->d_table);
    delete cb;
    return cuda_fail(e, "codebook upload");
  }
  *out = cb;
  return QP_OK;
}

void qp_codebook_free(qp_codebook* cb) {
  if (!cb) return;
  dev_free(cb->d_table);
  delete cb;
}

qp_status qp_rht_create(uint64_t seed, int d_in, int block, qp_rht** out) {
  if (!out) return fail(QP_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (d_in <= 0 || d_in % kTileCols) return fail(QP_ERR_DIM, "d_in=%d must be a positive multiple of 256", d_in);
  if (block == 0) block = d_in & (-d_in);   // largest power-of-two divisor (reading R9)
  if (block < 256 || (block & (block - 1)) || d_in % block || block > 32768)
    return fail(QP_ERR_DIM, "rotation block %d must be a power of two in [256, 32768] dividing d_in=%d", block, d_in);
  auto r = new qp_rht();
  r->seed = seed;
  r->d_in = d_in;
  r->block = block;
  r->sign_bits.assign((d_in + 31) / 32, 0u);
  for (int i = 0; i < d_in; ++i)
    if (splitmix64(seed, (uint64_t)i) >> 63) r->sign_bits[i >> 5] |= 1u << (i & 31);
  r->d_signs = static_cast<uint32_t*>(dev_alloc(r->sign_bits.size() * 4));
  if (!r->d_signs) {
    delete r;
    return fail(QP_ERR_ALLOC, "rotation allocation failed");
  }
  cudaError_t e = cudaMemcpy(r->d_signs, r->sign_bits.data(), r->sign_bits.size() * 4, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    dev_free(r->d_signs);
    delete r;
    return cuda_fail(e, "rotation upload");
  }
  *out = r;
  return QP_OK;
}

void qp_rht_free(qp_rht* r) {
  if (!r) return;
  dev_free(r->d_signs);
  delete r;
}

qp_status qp_rht_apply(const qp_rht* r, const void* x, qp_dtype xt, int batch, void* x_rot, void* stream) {
  if (!r || !x || !x_rot) return fail(QP_ERR_INVALID_ARG, "NULL argument to qp_rht_apply");
  if (batch < 1 || batch > 65535) return fail(QP_ERR_INVALID_ARG, "batch=%d", batch);
  if ((int)xt < 0 || (int)xt > 2) return fail(QP_ERR_INVALID_ARG, "bad dtype");
  return run_rht(r, x, xt, batch, static_cast<__half*>(x_rot), false, static_cast<cudaStream_t>(stream));
}

qp_status qp_layer_from_codes(const void* codes_host, size_t n_bytes, const float* scales_host, int d_out, int d_in,
                              qp_scheme scheme, int bits_x4, const qp_codebook* cb, const qp_rht* r, qp_layer** out) {
  if (!codes_host || !scales_host || !out || !r) return fail(QP_ERR_INVALID_ARG, "NULL argument to qp_layer_from_codes");
  *out = nullptr;
  qp_status st = check_shape(scheme, bits_x4, d_out, d_in);
  if (st != QP_OK) return st;
  if ((st = check_codebook(cb, scheme, bits_x4)) != QP_OK) return st;
  if (r->d_in != d_in) return fail(QP_ERR_CONFIG_MISMATCH, "rotation is for d_in=%d, layer has %d", r->d_in, d_in);
  const size_t need = layout_bytes(scheme, bits_x4, d_out, d_in);
  if (n_bytes != need)
    return fail(QP_ERR_LENGTH, "codes must be exactly %zu bytes (d_out*d_in*bits/8, LAYOUT.md), got %zu", need, n_bytes);
  auto l = new qp_layer();
  if ((st = layer_init(l, d_out, d_in, scheme, bits_x4, cb, r)) != QP_OK) {
    layer_release(l);
    delete l;
    return st;
  }
  cudaError_t e = cudaMemcpy(l->d_codes, codes_host, need, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(l->d_scales, scales_host, (size_t)d_out * 4, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    layer_release(l);
    delete l;
    return cuda_fail(e, "layer upload");
  }
  *out = l;
  return QP_OK;
}

qp_status qp_layer_get_codes(const qp_layer* l, void* codes_host, size_t n_bytes) {
  if (!l || !codes_host) return fail(QP_ERR_INVALID_ARG, "NULL argument");
  if (n_bytes != l->code_bytes) return fail(QP_ERR_LENGTH, "layer holds %zu code bytes", l->code_bytes);
  CUDA_TRY(cudaMemcpy(codes_host, l->d_codes, n_bytes, cudaMemcpyDeviceToHost), "codes download");
  return QP_OK;
}

qp_status qp_layer_get_scales(const qp_layer* l, float* scales_host) {
  if (!l || !scales_host) return fail(QP_ERR_INVALID_ARG, "NULL argument");
  CUDA_TRY(cudaMemcpy(scales_host, l->d_scales, (size_t)l->d_out * 4, cudaMemcpyDeviceToHost), "scales download");
  return QP_OK;
}

qp_status qp_layer_info(const qp_layer* l, size_t* code_bytes, double* bits_per_weight, int* d_out, int* d_in) {
  if (!l) return fail(QP_ERR_INVALID_ARG, "layer is NULL");
  if (code_bytes) *code_bytes = l->code_bytes;
  if (bits_per_weight) *bits_per_weight = 8.0 * (double)l->code_bytes / ((double)l->d_out * l->d_in);
  if (d_out) *d_out = l->d_out;
  if (d_in) *d_in = l->d_in;
  return QP_OK;
}

void qp_layer_free(qp_layer* l) {
  if (!l) return;
  layer_release(l);
  delete l;
}

qp_status qp_linear_fwd(const qp_layer* l, const void* x, qp_dtype xt, int batch, void* y, qp_dtype yt,
                        unsigned flags, void* stream) {
  if (!l || !y) return fail(QP_ERR_INVALID_ARG, "NULL layer or y");
  qp_status st = check_fwd_args(x, xt, batch, yt, flags);
  if (st != QP_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool pdl = !(flags & QP_NO_PDL) && !pdl_disabled_by_env();
  const __half* xr = static_cast<const __half*>(x);
  void* ys[1] = {y};
  // fp32 output: the preceding kernel (rotation, or a zeroing kernel) zeroes y and CTAs that share
  // a row tile add into it; fp16 output: the same into the layer's fp32 workspace, the warp that
  // completes a row tile converting it; QP_DETERMINISTIC: in-order cross-CTA reduction instead
  const bool ws16 = yt == QP_F16 && !(flags & QP_DETERMINISTIC) && !g_peer_out && !f16_inorder_by_env();
  const bool atomic = (yt == QP_F32 && !(flags & QP_DETERMINISTIC)) || ws16;
  const long long zn[1] = {(long long)batch * l->d_out};
  const int rtb[2] = {0, l->d_out / kTileRows};
  const int ldy[1] = {l->d_out};
  void* zs[1] = {ws16 ? static_cast<void*>(l->d_yws) : y};
  if (!(flags & QP_X_PREROTATED) && !ws16 && ((flags & QP_FUSE_RHT) || fused_rht_by_env())) {
    // one kernel: every CTA rotates x itself (and zeroes y) -- no rotation kernel on the path;
    // falls through to the two-kernel path when x' does not fit the fused plan
    const FusedRot fr{l->rht, x, xt, atomic && !(flags & QP_Y_ACCUMULATE)};
    bool unsup = false;
    st = run_gemv(l, nullptr, batch, 1, rtb, ys, ldy, yt, pdl, s, atomic, 0, &fr, &unsup, (flags & QP_Y_ACCUMULATE) != 0);
    if (st != QP_OK || !unsup) return st;
  }
  int side = 0;
  if (!(flags & QP_X_PREROTATED)) {
    const int nz = atomic && !(flags & QP_Y_ACCUMULATE) ? 1 : 0;
    if ((st = run_rht(l->rht, x, xt, batch, l->d_xrot, pdl, s, nz, zs, zn)) != QP_OK) return st;
    xr = l->d_xrot;
    side = batch * (l->d_in / l->rht->block);
  } else if (atomic && !(flags & QP_Y_ACCUMULATE)) {
    RhtParams zp{};
    zp.n_zero = 1;
    zp.zero_ptr[0] = static_cast<float*>(zs[0]);
    zp.zero_n[0] = zn[0];
    side = zero_ctas(zn, 1);
    cudaError_t e = launch_zero(zp, side, pdl, s);
    if (e != cudaSuccess) return cuda_fail(e, "zero kernel launch");
  }
  return run_gemv(l, xr, batch, 1, rtb, ys, ldy, yt, pdl, s, atomic, side, nullptr, nullptr,
                  (flags & QP_Y_ACCUMULATE) != 0);
}

qp_status qp_dequantize(const qp_layer* l, void* W_hat_fp16, void* stream) {
  if (!l || !W_hat_fp16) return fail(QP_ERR_INVALID_ARG, "NULL argument to qp_dequantize");
  GemvParams p{};
  p.codes = l->d_codes;
  p.scales = l->d_scales;
  p.table = l->cb->d_table;
  p.table_words = l->cb->table_words;
  p.RT = l->d_out / kTileRows;
  p.KT = l->d_in / kTileCols;
  p.d_in = l->d_in;
  p.batch = 1;
  p.w_out = static_cast<__half*>(W_hat_fp16);
  set_magics(p, l->grid);
  cudaError_t e = l->launcher(p, l->grid, 0, true, false, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "dequantize launch");
  count_launch();
  return QP_OK;
}

qp_status qp_fuse(const qp_layer* const* members, int n, qp_group** out) {
  if (!members || !out || n < 1) return fail(QP_ERR_INVALID_ARG, "bad arguments to qp_fuse");
  *out = nullptr;
  if (n > kMaxGroup) return fail(QP_ERR_INVALID_ARG, "at most %d members per group", kMaxGroup);
  const qp_layer* m0 = members[0];
  int d_out = 0;
  for (int i = 0; i < n; ++i) {
    const qp_layer* m = members[i];
    if (!m) return fail(QP_ERR_INVALID_ARG, "member %d is NULL", i);
    if (m->d_in != m0->d_in || m->rht != m0->rht || m->scheme != m0->scheme || m->bits_x4 != m0->bits_x4 ||
        m->cb != m0->cb)
      return fail(QP_ERR_CONFIG_MISMATCH, "fused members must share d_in, rotation, scheme, width and codebook (P:470)");
    d_out += m->d_out;
  }
  auto g = new qp_group();
  g->cat = new qp_layer();
  qp_status st = layer_init(g->cat, d_out, m0->d_in, m0->scheme, m0->bits_x4, m0->cb, m0->rht);
  if (st != QP_OK) {
    qp_group_free(g);
    return st;
  }
  size_t off = 0;
  int row = 0;
  for (int i = 0; i < n; ++i) {
    const qp_layer* m = members[i];
    cudaError_t e = cudaMemcpy(g->cat->d_codes + off, m->d_codes, m->code_bytes, cudaMemcpyDeviceToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(g->cat->d_scales + row, m->d_scales, (size_t)m->d_out * 4, cudaMemcpyDeviceToDevice);
    if (e != cudaSuccess) {
      qp_group_free(g);
      return cuda_fail(e, "group concatenation");
    }
    off += m->code_bytes;
    row += m->d_out;
    g->d_outs.push_back(m->d_out);
  }
  // device-to-device copies on the legacy stream: complete before the group is used elsewhere
  if (cudaError_t e = cudaStreamSynchronize(0); e != cudaSuccess) {
    qp_group_free(g);
    return cuda_fail(e, "group concatenation");
  }
  *out = g;
  return QP_OK;
}

void qp_group_free(qp_group* g) {
  if (!g) return;
  if (g->cat) {
    layer_release(g->cat);
    delete g->cat;
  }
  delete g;
}

qp_status qp_fused_linear(const qp_group* g, const void* x, qp_dtype xt, int batch, void* const* ys, qp_dtype yt,
                          unsigned flags, void* stream) {
  if (!g || !ys) return fail(QP_ERR_INVALID_ARG, "NULL group or ys");
  qp_status st = check_fwd_args(x, xt, batch, yt, flags);
  if (st != QP_OK) return st;
  const int n = (int)g->d_outs.size();
  for (int i = 0; i < n; ++i)
    if (!ys[i]) return fail(QP_ERR_INVALID_ARG, "ys[%d] is NULL", i);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const qp_layer* l = g->cat;
  const __half* xr = static_cast<const __half*>(x);
  if (pdl_disabled_by_env()) flags |= QP_NO_PDL;
  const bool ws16 = yt == QP_F16 && !(flags & QP_DETERMINISTIC) && !f16_inorder_by_env();
  const bool atomic = (yt == QP_F32 && !(flags & QP_DETERMINISTIC)) || ws16;
  long long zn[kMaxGroup];
  for (int i = 0; i < n; ++i) zn[i] = (long long)batch * g->d_outs[i];
  void* zs[kMaxGroup];
  {
    size_t off = 0;
    for (int i = 0; i < n; ++i) {
      zs[i] = ws16 ? static_cast<void*>(l->d_yws + off) : ys[i];
      off += (size_t)batch * g->d_outs[i];
    }
  }
  int rtb[kMaxGroup + 1];
  int ldy[kMaxGroup];
  rtb[0] = 0;
  for (int i = 0; i < n; ++i) {
    rtb[i + 1] = rtb[i] + g->d_outs[i] / kTileRows;
    ldy[i] = g->d_outs[i];
  }
  if (!(flags & QP_X_PREROTATED) && !ws16 && ((flags & QP_FUSE_RHT) || fused_rht_by_env())) {
    const FusedRot fr{l->rht, x, xt, atomic && !(flags & QP_Y_ACCUMULATE)};
    bool unsup = false;
    st = run_gemv(l, nullptr, batch, n, rtb, ys, ldy, yt, !(flags & QP_NO_PDL), s, atomic, 0, &fr, &unsup,
                  (flags & QP_Y_ACCUMULATE) != 0);
    if (st != QP_OK || !unsup) return st;
  }
  int side = 0;
  if (!(flags & QP_X_PREROTATED)) {
    const int nz = atomic && !(flags & QP_Y_ACCUMULATE) ? n : 0;
    if ((st = run_rht(l->rht, x, xt, batch, l->d_xrot, !(flags & QP_NO_PDL), s, nz, zs, zn)) != QP_OK) return st;
    xr = l->d_xrot;
    side = batch * (l->d_in / l->rht->block);
  } else if (atomic && !(flags & QP_Y_ACCUMULATE)) {
    RhtParams zp{};
    zp.n_zero = n;
    for (int i = 0; i < n; ++i) {
      zp.zero_ptr[i] = static_cast<float*>(zs[i]);
      zp.zero_n[i] = zn[i];
    }
    side = zero_ctas(zn, n);
    cudaError_t e = launch_zero(zp, side, !(flags & QP_NO_PDL), s);
    if (e != cudaSuccess) return cuda_fail(e, "zero kernel launch");
  }
  return run_gemv(l, xr, batch, n, rtb, ys, ldy, yt, !(flags & QP_NO_PDL), s, atomic, side, nullptr, nullptr,
                  (flags & QP_Y_ACCUMULATE) != 0);
}

qp_status qp_shard_range(int d_out, int d_in, qp_scheme scheme, int bits_x4, int rank, int world, int* row0,
                         int* rows, size_t* byte0, size_t* nbytes) {
  if (!row0 || !rows || !byte0 || !nbytes) return fail(QP_ERR_INVALID_ARG, "NULL output pointer to qp_shard_range");
  if (world < 1 || rank < 0 || rank >= world) return fail(QP_ERR_INVALID_ARG, "rank %d / world %d", rank, world);
  if (!width_ok(scheme, bits_x4)) return fail(QP_ERR_UNSUPPORTED_WIDTH, "unsupported width %.2f", bits_x4 / 4.0);
  qp_status st = check_shape(scheme, bits_x4, d_out, d_in);
  if (st != QP_OK) return st;
  if (d_out % world || (d_out / world) % kTileRows)
    return fail(QP_ERR_PARTITION_MISMATCH, "d_out=%d does not split into %d row blocks of a multiple of 32", d_out,
                world);
  const int m = d_out / world;
  const size_t shard_bytes = layout_bytes(scheme, bits_x4, m, d_in);
  *row0 = rank * m;
  *rows = m;
  *byte0 = (size_t)rank * shard_bytes;
  *nbytes = shard_bytes;
  return QP_OK;
}

qp_status qp_layer_shard(const qp_layer* l, int rank, int world, qp_layer** out) {
  if (!l || !out) return fail(QP_ERR_INVALID_ARG, "NULL argument to qp_layer_shard");
  *out = nullptr;
  int row0 = 0, m = 0;
  size_t byte0 = 0, nb = 0;
  qp_status rs = qp_shard_range(l->d_out, l->d_in, l->scheme, l->bits_x4, rank, world, &row0, &m, &byte0, &nb);
  if (rs != QP_OK) return rs;
  auto s = new qp_layer();
  qp_status st = layer_init(s, m, l->d_in, l->scheme, l->bits_x4, l->cb, l->rht);
  if (st != QP_OK) {
    layer_release(s);
    delete s;
    return st;
  }
  // row-tile-major storage: rows [rank*m, (rank+1)*m) are one contiguous byte range (LAYOUT.md)
  cudaError_t e = cudaMemcpy(s->d_codes, l->d_codes + byte0, nb, cudaMemcpyDeviceToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(s->d_scales, l->d_scales + row0, (size_t)m * 4, cudaMemcpyDeviceToDevice);
  if (e == cudaSuccess) e = cudaStreamSynchronize(0);   // legacy-stream copies done before use
  if (e == cudaSuccess) {
    // the all-gather scratch of qp_linear_fwd_sharded for up to batch 8, fp32: allocated here, so the
    // forward never allocates (CUDA-graph capture safe)
    s->gather_bytes = (size_t)(world + 1) * 8 * m * 4;
    s->d_gather = dev_alloc(s->gather_bytes);
    if (!s->d_gather) {
      layer_release(s);
      delete s;
      return fail(QP_ERR_ALLOC, "shard all-gather scratch allocation failed");
    }
  }
  if (e != cudaSuccess) {
    layer_release(s);
    delete s;
    return cuda_fail(e, "shard copy");
  }
  *out = s;
  return QP_OK;
}

qp_status qp_nccl_unique_id(void* id128) {
  if (!id128) return fail(QP_ERR_INVALID_ARG, "id buffer is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclResult_t r = ncclGetUniqueId(static_cast<ncclUniqueId*>(id128));
  if (r != ncclSuccess) return fail(QP_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  return QP_OK;
}

qp_status qp_nccl_comm_create(const void* id128, int world, int rank, void** comm) {
  if (!id128 || !comm) return fail(QP_ERR_INVALID_ARG, "NULL argument");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclComm_t c = nullptr;
  ncclResult_t r = ncclCommInitRank(&c, world, id, rank);
  if (r != ncclSuccess) return fail(QP_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  *comm = c;
  return QP_OK;
}

qp_status qp_nccl_comm_destroy(void* comm) {
  if (!comm) return QP_OK;
  ncclResult_t r = ncclCommDestroy(static_cast<ncclComm_t>(comm));
  if (r != ncclSuccess) return fail(QP_ERR_NCCL, "ncclCommDestroy: %s", ncclGetErrorString(r));
  return QP_OK;
}

qp_status qp_linear_fwd_sharded(const qp_layer* shard, const void* x, qp_dtype xt, int batch, void* y_full,
                                qp_dtype yt, void* comm, unsigned flags, void* stream) {
  if (!shard || !y_full || !comm) return fail(QP_ERR_INVALID_ARG, "NULL argument to qp_linear_fwd_sharded");
  qp_status st = check_fwd_args(x, xt, batch, yt, flags);
  if (st != QP_OK) return st;
  if (flags & QP_Y_ACCUMULATE)
    return fail(QP_ERR_INVALID_ARG, "qp_linear_fwd_sharded: QP_Y_ACCUMULATE is not supported (the all-gather "
                "overwrites y_full). Remedy: add the residual after the call");
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  int world = 0;
  if (ncclCommCount(c, &world) != ncclSuccess || world < 1) return fail(QP_ERR_NCCL, "ncclCommCount failed");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int m = shard->d_out;
  const int eb = yt == QP_F32 ? 4 : 2;
  qp_layer* l = const_cast<qp_layer*>(shard);
  const size_t need = (size_t)(world + 1) * batch * m * eb;
  if (l->gather_bytes < need)
    return fail(QP_ERR_CONFIG_MISMATCH, "qp_linear_fwd_sharded: the layer is not a shard of a %d-rank split "
                "(qp_layer_shard allocates the all-gather scratch). Remedy: shard with world = %d", world, world);
  uint8_t* local = static_cast<uint8_t*>(l->d_gather);              // [batch][m]
  uint8_t* gathered = local + (size_t)batch * m * eb;                // [world][batch][m]
  if ((st = qp_linear_fwd(shard, x, xt, batch, local, yt, flags, stream)) != QP_OK) return st;
  void* recv = batch == 1 ? y_full : gathered;
  ncclResult_t r = ncclAllGather(local, recv, (size_t)batch * m, yt == QP_F32 ? ncclFloat32 : ncclFloat16, c, s);
  if (r != ncclSuccess) return fail(QP_ERR_NCCL, "ncclAllGather: %s", ncclGetErrorString(r));
  if (batch > 1) {
    cudaError_t e = launch_gather_permute(gathered, y_full, world, batch, m, eb, s);
    if (e != cudaSuccess) return cuda_fail(e, "gather permute");
  }
  ncclResult_t ae = ncclSuccess;   // asynchronous NCCL faults of earlier calls surface here
  if (ncclCommGetAsyncError(c, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress)
    return fail(QP_ERR_NCCL, "asynchronous NCCL error: %s", ncclGetErrorString(ae));
  return QP_OK;
}

}  // extern "C"

// accessors for qp_offline.cpp (not part of the public ABI)
extern "C" qp_status qp_linear_fwd_sharded_p2p(const qp_layer* shard, const void* x, qp_dtype xt, int batch,
                                               void* const* y_peers, unsigned* const* flag_peers, int rank,
                                               int world, qp_dtype yt, unsigned flags, void* stream) {
  if (!shard || !y_peers || !flag_peers) return fail(QP_ERR_INVALID_ARG, "NULL argument to qp_linear_fwd_sharded_p2p");
  if (world < 1 || world > kMaxGroup || rank < 0 || rank >= world)
    return fail(QP_ERR_INVALID_ARG, "rank %d / world %d (1..%d ranks)", rank, world, kMaxGroup);
  for (int k = 0; k < world; ++k)
    if (!y_peers[k] || !flag_peers[k]) return fail(QP_ERR_INVALID_ARG, "peer %d pointer is NULL", k);
  if (flags & (QP_Y_ACCUMULATE | QP_FUSE_RHT))
    return fail(QP_ERR_INVALID_ARG, "qp_linear_fwd_sharded_p2p: QP_Y_ACCUMULATE / QP_FUSE_RHT not supported");
  // round entry barrier: no rank stores round n into a peer's y_full before that peer has entered
  // round n (its stream-ordered readers of round n-1 are done)
  if (cudaError_t e = launch_peer_enter(flag_peers, rank, world, static_cast<cudaStream_t>(stream)); e != cudaSuccess)
    return cuda_fail(e, "peer enter kernel launch");
  // every final value is written once, by its owner, to every rank: the in-order epilogue
  const PeerOut po{world, rank, rank * shard->d_out, world * shard->d_out, y_peers, flag_peers};
  g_peer_out = &po;
  const qp_status st = qp_linear_fwd(shard, x, xt, batch, y_peers[rank], yt, flags | QP_DETERMINISTIC, stream);
  g_peer_out = nullptr;
  if (st != QP_OK) return st;
  cudaError_t e = launch_peer_wait(flag_peers[rank], world, static_cast<cudaStream_t>(stream), 1);
  if (e != cudaSuccess) return cuda_fail(e, "peer wait kernel launch");
  return QP_OK;
}

extern "C" qp_status qp_gather_permute(const void* src, void* dst, int world, int batch, int m, int elem_bytes,
                                       void* stream) {
  if (!src || !dst) return fail(QP_ERR_INVALID_ARG, "NULL argument to qp_gather_permute");
  if (world < 1 || batch < 1 || m < 1 || (elem_bytes != 2 && elem_bytes != 4))
    return fail(QP_ERR_INVALID_ARG, "qp_gather_permute: world %d batch %d m %d elem_bytes %d", world, batch, m,
                elem_bytes);
  cudaError_t e = launch_gather_permute(src, dst, world, batch, m, elem_bytes, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "gather permute");
  return QP_OK;
}

namespace {
// cuMemGetAddressRange through the runtime's driver entry point (no link-time libcuda dependency):
// base and size of the allocation containing ptr. IPC handles name whole allocations, and PyTorch's
// caching allocator (or qp_set_allocator) hands out pointers inside larger segments.
using AddrRangeFn = int (*)(unsigned long long*, size_t*, unsigned long long);
cudaError_t alloc_base(const void* ptr, uintptr_t* base) {
  static AddrRangeFn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q);
    if (e != cudaSuccess || !f) return e != cudaSuccess ? e : cudaErrorNotSupported;
    fn = reinterpret_cast<AddrRangeFn>(f);
  }
  unsigned long long b = 0;
  size_t n = 0;
  if (fn(&b, &n, (unsigned long long)reinterpret_cast<uintptr_t>(ptr)) != 0) return cudaErrorInvalidValue;
  *base = (uintptr_t)b;
  return cudaSuccess;
}
}  // namespace

extern "C" qp_status qp_ipc_handle(const void* dev_ptr, void* handle72) {
  if (!dev_ptr || !handle72) return fail(QP_ERR_INVALID_ARG, "NULL argument to qp_ipc_handle");
  uintptr_t base = 0;
  cudaError_t e = alloc_base(dev_ptr, &base);
  if (e != cudaSuccess) return cuda_fail(e, "cuMemGetAddressRange");
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  const uint64_t off = (uint64_t)(reinterpret_cast<uintptr_t>(dev_ptr) - base);
  std::memcpy(handle72, &h, 64);
  std::memcpy(static_cast<uint8_t*>(handle72) + 64, &off, 8);
  return QP_OK;
}

extern "C" qp_status qp_ipc_open(const void* handle72, void** dev_ptr) {
  if (!dev_ptr || !handle72) return fail(QP_ERR_INVALID_ARG, "NULL argument to qp_ipc_open");
  cudaIpcMemHandle_t h;
  uint64_t off = 0;
  std::memcpy(&h, handle72, 64);
  std::memcpy(&off, static_cast<const uint8_t*>(handle72) + 64, 8);
  void* base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
  *dev_ptr = static_cast<uint8_t*>(base) + off;
  return QP_OK;
}

extern "C" qp_status qp_ipc_close(void* dev_ptr) {
  uintptr_t base = 0;
  cudaError_t e = alloc_base(dev_ptr, &base);
  if (e == cudaSuccess) e = cudaIpcCloseMemHandle(reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
  return QP_OK;
}

extern "C" qp_status qp_codebook_set_scale(qp_codebook* cb, double alpha) {
  if (!cb) return fail(QP_ERR_INVALID_ARG, "codebook is NULL");
  if (!(alpha > 0.0) || !std::isfinite(alpha))
    return fail(QP_ERR_INVALID_ARG, "alpha=%g must be positive and finite (codebooks/tcq_alpha.json)", alpha);
  cb->alpha = alpha;
  return QP_OK;
}

extern "C" qp_status qp_internal_codebook_alpha(const qp_codebook* cb, double* alpha) {
  if (!cb || !alpha) return fail(QP_ERR_INVALID_ARG, "NULL argument");
  *alpha = cb->alpha;
  return QP_OK;
}

extern "C" qp_status qp_internal_codebook_info(const qp_codebook* cb, int* L, int* tb, const uint16_t** host,
                                               size_t* n) {
  if (!cb) return fail(QP_ERR_INVALID_ARG, "codebook is NULL");
  *L = cb->L;
  *tb = cb->tb;
  *host = cb->host.data();
  *n = cb->host.size();
  return QP_OK;
}
extern "C" qp_status qp_internal_rht_info(const qp_rht* r, uint64_t* seed, int* d_in, int* block,
                                          const uint32_t** sign_bits) {
  if (!r) return fail(QP_ERR_INVALID_ARG, "rotation is NULL");
  *seed = r->seed;
  *d_in = r->d_in;
  *block = r->block;
  *sign_bits = r->sign_bits.data();
  return QP_OK;
}

// ---------------------------------------------------------------------------------------
// persistent multi-layer engine (qp_multi_*; kernel: qp_engine.cuh)
// ---------------------------------------------------------------------------------------
struct qp_multi {
  struct Group {
    int first = 0, n = 0;
    EngineLauncher launch = nullptr;   // nullptr: per-layer qp_linear_fwd (no engine variant)
    unsigned* d_gen = nullptr;         // [2] exit counter, launches completed
  };
  std::vector<const qp_layer*> layers;
  std::vector<Group> groups;
  std::vector<__half*> d_xr;           // per layer: x' [8][d_in]
  std::vector<float*> d_ws;            // per layer: [8][d_out] fp32, zero between launches
  std::vector<int*> d_cnt;             // per layer: [RT] k-tile counters, zero between launches
  unsigned* d_flags = nullptr;         // per layer: ready, kFlagStride words apart (own L2 slice)
  unsigned* d_gens = nullptr;          // per group [8]: exit counter, pad, 64-bit entry / exit counts
};

namespace {
bool same_table(const qp_codebook* a, const qp_codebook* b) {
  return a == b || (a->mode == b->mode && a->L == b->L && a->tb == b->tb && a->reps == b->reps &&
                    a->table_words == b->table_words && a->host == b->host);
}
bool eng_single() {   // QP_ENG_SINGLE=0: one-layer groups through the per-layer path (experiments)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("QP_ENG_SINGLE");
    v = e ? (atoi(e) != 0 ? 1 : 0) : 1;
  }
  return v == 1;
}
int eng_rp_min_batch() {   // QP_ENG_RP2_MIN_BATCH: smallest batch for row-pair units (9 = never)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("QP_ENG_RP2_MIN_BATCH");
    v = e ? atoi(e) : 8;
  }
  return v;
}
int eng_late_stages() {   // QP_ENG_LATE=1: fill ring stages 1.. only once x' is ready (experiment)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("QP_ENG_LATE");
    v = e ? atoi(e) : 0;
  }
  return v;
}
double eng_row_cost() {   // QP_ENG_ROWCOST: per-row-tile overhead of a layer, in tiles (CTA range balance)
  static double v = -1;
  if (v < 0) {
    const char* e = getenv("QP_ENG_ROWCOST");
    v = e ? atof(e) : 0.0;
  }
  return v;
}
double eng_half_cost() {   // QP_ENG_HALFCOST: extra cost of a half-TCQ tile (two width runs per row)
  static double v = -1;
  if (v < 0) {
    const char* e = getenv("QP_ENG_HALFCOST");
    v = e ? atof(e) : 0.0;
  }
  return v;
}
double eng_job_tiles(int batch) {   // QP_ENG_JOB_TILES: tiles of GEMV work one rotation job displaces
  // A job (one Hadamard block of one batch row) costs about as much as 16 tiles at batch 1; a tile's
  // cost grows with the batch (8 activation rows per MMA, x' loads), so fewer tiles per job above it:
  // 16 * 8 / (7 + batch) = 16 at batch 1, 8.5 at batch 8 (A/B: batch 8 -2 to -6 %, profiles/r2/v5/job_tiles_ab.txt)
  static double v = -2;
  if (v == -2) {
    const char* e = getenv("QP_ENG_JOB_TILES");
    v = e ? atof(e) : -1.0;
  }
  return v >= 0 ? v : 16.0 * 8.0 / (7.0 + batch);
}
void multi_release(qp_multi* m) {
  for (auto p : m->d_xr) dev_free(p);
  for (auto p : m->d_ws) dev_free(p);
  for (auto p : m->d_cnt) dev_free(p);
  dev_free(m->d_flags);
  dev_free(m->d_gens);
}
}  // namespace

extern "C" qp_status qp_multi_create(const qp_layer* const* layers, int n, qp_multi** out) {
  if (!layers || !out || n < 1) return fail(QP_ERR_INVALID_ARG, "bad arguments to qp_multi_create");
  *out = nullptr;
  for (int i = 0; i < n; ++i)
    if (!layers[i]) return fail(QP_ERR_INVALID_ARG, "layer %d is NULL", i);
  auto m = new qp_multi();
  m->layers.assign(layers, layers + n);
  // consecutive layers sharing a decode table (and an engine variant covering their step widths)
  // form one persistent launch; at most kMaxEngOps layers each
  for (int i = 0; i < n;) {
    qp_multi::Group gr;
    gr.first = i;
    int cmin = layers[i]->c_lo, cmax = layers[i]->c_hi;
    const qp_codebook* cb = layers[i]->cb;
    EngineLauncher f = find_engine(cb->mode, cb->mode == DEC_LUT2 || cb->mode == DEC_SCALAR ? 0 : cb->L,
                                   cb->mode == DEC_LUT2 ? 0 : cb->tb, cb->reps, cmin, cmax);
    int j = i + 1;
    if (f) {
      while (j < n && j - i < kMaxEngOps && same_table(layers[j]->cb, cb)) {
        const int lo = std::min(cmin, layers[j]->c_lo), hi = std::max(cmax, layers[j]->c_hi);
        EngineLauncher f2 = find_engine(cb->mode, cb->mode == DEC_LUT2 || cb->mode == DEC_SCALAR ? 0 : cb->L,
                                        cb->mode == DEC_LUT2 ? 0 : cb->tb, cb->reps, lo, hi);
        if (!f2) break;
        f = f2;
        cmin = lo;
        cmax = hi;
        ++j;
      }
    }
    gr.n = j - i;
    // (QP_ENG_SINGLE=0: one-layer groups through the per-layer path instead -- faster for one layer
    // launched back to back, slower inside a mixed sequence such as C5: profiles/r2/one_layer.md)
    gr.launch = (gr.n == 1 && !eng_single()) ? nullptr : f;
    m->groups.push_back(gr);
    i = j;
  }
  m->d_flags = static_cast<unsigned*>(dev_alloc((size_t)kFlagStride * n * 4));
  m->d_gens = static_cast<unsigned*>(dev_alloc(m->groups.size() * 8 * 4));
  bool ok = m->d_flags && m->d_gens;
  for (int i = 0; i < n && ok; ++i) {
    const qp_layer* l = layers[i];
    m->d_xr.push_back(static_cast<__half*>(dev_alloc((size_t)8 * l->d_in * 2)));
    m->d_ws.push_back(static_cast<float*>(dev_alloc((size_t)8 * l->d_out * 4)));
    m->d_cnt.push_back(static_cast<int*>(dev_alloc((size_t)(l->d_out / kTileRows) * 4)));
    ok = m->d_xr.back() && m->d_ws.back() && m->d_cnt.back();
    if (ok && (cudaMemset(m->d_ws.back(), 0, (size_t)8 * l->d_out * 4) != cudaSuccess ||
               cudaMemset(m->d_cnt.back(), 0, (size_t)(l->d_out / kTileRows) * 4) != cudaSuccess))
      ok = false;
  }
  if (ok && (cudaMemset(m->d_flags, 0, (size_t)kFlagStride * n * 4) != cudaSuccess ||
             cudaMemset(m->d_gens, 0, m->groups.size() * 8 * 4) != cudaSuccess))
    ok = false;
  // the memsets run on the legacy stream: complete them before any stream uses the object
  if (ok && cudaDeviceSynchronize() != cudaSuccess) ok = false;
  if (!ok) {
    multi_release(m);
    delete m;
    return fail(QP_ERR_ALLOC, "qp_multi_create: device allocation failed");
  }
  for (size_t k = 0; k < m->groups.size(); ++k) m->groups[k].d_gen = m->d_gens + 8 * k;   // 8-byte aligned
  *out = m;
  return QP_OK;
}

extern "C" void qp_multi_free(qp_multi* m) {
  if (!m) return;
  multi_release(m);
  delete m;
}

extern "C" qp_status qp_multi_info(const qp_multi* m, int* n_layers, int* n_launches, int* n_engine_launches) {
  if (!m) return fail(QP_ERR_INVALID_ARG, "NULL qp_multi");
  if (n_layers) *n_layers = (int)m->layers.size();
  if (n_launches) *n_launches = (int)m->groups.size();
  if (n_engine_launches) {
    int k = 0;
    for (const auto& g : m->groups) k += g.launch ? 1 : 0;
    *n_engine_launches = k;
  }
  return QP_OK;
}

namespace {
// fused all-gather destinations of qp_multi_fwd_sharded_p2p
struct EngPeers {
  int world, rank;
  void* const* y;              // [n_layers * world]
  unsigned* const* flag;       // [world]
};

qp_status multi_fwd_impl(qp_multi* m, const void* const* xs, qp_dtype xt, int batch, void* const* ys, qp_dtype yt,
                         unsigned flags, void* stream, const EngPeers* peers);
}  // namespace

extern "C" qp_status qp_multi_fwd(qp_multi* m, const void* const* xs, qp_dtype xt, int batch, void* const* ys,
                                  qp_dtype yt, unsigned flags, void* stream) {
  if (!m || !xs || !ys) return fail(QP_ERR_INVALID_ARG, "NULL argument to qp_multi_fwd");
  return multi_fwd_impl(m, xs, xt, batch, ys, yt, flags, stream, nullptr);
}

namespace {
qp_status multi_fwd_impl(qp_multi* m, const void* const* xs, qp_dtype xt, int batch, void* const* ys, qp_dtype yt,
                         unsigned flags, void* stream, const EngPeers* peers) {
  const int n = (int)m->layers.size();
  for (int i = 0; i < n; ++i) {
    if (!ys[i]) return fail(QP_ERR_INVALID_ARG, "ys[%d] is NULL", i);
    qp_status st = check_fwd_args(xs[i], xt, batch, yt, flags);
    if (st != QP_OK) return st;
    if (!(flags & QP_X_PREROTATED) && (reinterpret_cast<uintptr_t>(xs[i]) & 15u))
      return fail(QP_ERR_INVALID_ARG, "xs[%d] must be 16-byte aligned (vector loads of the rotation)", i);
  }
  if (flags & (QP_DETERMINISTIC | QP_FUSE_RHT))
    return fail(QP_ERR_INVALID_ARG, "qp_multi_fwd: QP_DETERMINISTIC / QP_FUSE_RHT are per-layer options (use "
                "qp_linear_fwd)");
  const unsigned layer_flags = flags & ~QP_INDEPENDENT;   // the per-layer fallback ignores QP_INDEPENDENT
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool pdl = !(flags & QP_NO_PDL) && !pdl_disabled_by_env();
  const bool pre = (flags & QP_X_PREROTATED) != 0;
  for (const auto& gr : m->groups) {
    if (!gr.launch) {
      if (peers)
        return fail(QP_ERR_UNSUPPORTED, "qp_multi_fwd_sharded_p2p: layer %d has no engine variant (the fused "
                    "all-gather runs in the engine epilogue). Remedy: qp_linear_fwd_sharded_p2p per layer",
                    gr.first);
      for (int i = gr.first; i < gr.first + gr.n; ++i) {
        qp_status st = qp_linear_fwd(m->layers[i], xs[i], xt, batch, ys[i], yt, layer_flags, stream);
        if (st != QP_OK) return st;
      }
      continue;
    }
    static thread_local EngParams p;   // ~6 KB: not on the stack
    std::memset(&p, 0, sizeof p);
    p.n_ops = gr.n;
    p.batch = batch;
    p.x_dtype = (int)xt;
    p.y_f32 = yt == QP_F32 ? 1 : 0;
    p.y_accum = (flags & QP_Y_ACCUMULATE) ? 1 : 0;
    p.table = m->layers[gr.first]->cb->d_table;
    p.gen = gr.d_gen;
    // row-pair units (two row tiles per k tile share the activation fragments) from batch 4 on,
    // when every layer of the launch has an even number of row tiles
    // -- and only with >= 8 row-pair units per warp: coarser units cost balance on small launches
    // (C3's three layers per launch: +7% at batch 4; the 9-layer sets: -9% at batch 8; ab_rp.md)
    int rp = batch >= eng_rp_min_batch() && m->layers[gr.first]->cb->mode == DEC_LUT2 ? 2 : 1;
    {
      long long tiles_all = 0;
      for (int k = 0; k < gr.n; ++k) {
        const qp_layer* l = m->layers[gr.first + k];
        if ((l->d_out / kTileRows) % 2) rp = 1;
        tiles_all += (long long)(l->d_out / kTileRows) * (l->d_in / kTileCols);
      }
      if (tiles_all / 2 < 8LL * 16 * std::min(num_sms(), kMaxEngCtas)) rp = 1;
    }
    p.rp = rp;
    uint32_t tiles = 0;
    int jobs = 0, scratch = 0;
    for (int k = 0; k < gr.n; ++k) {
      const int i = gr.first + k;
      const qp_layer* l = m->layers[i];
      EngOp& o = p.op[k];
      o.codes = l->d_codes;
      o.scales = l->d_scales;
      o.RT = l->d_out / kTileRows;
      o.KT = l->d_in / kTileCols;
      o.KH = o.KT / 2;
      o.c_lo = l->c_lo;
      o.c_hi = l->c_hi;
      o.rowtile_bytes = (long long)o.KH * 512 * o.c_lo + (long long)(o.KT - o.KH) * 512 * o.c_hi;
      o.d_in = l->d_in;
      o.d_out = l->d_out;
      o.tile0 = tiles;
      tiles += (uint32_t)((o.RT / rp) * o.KT);
      o.x_raw = xs[i];
      o.xr = pre ? static_cast<__half*>(const_cast<void*>(xs[i])) : m->d_xr[i];
      o.rht_signs = l->rht->d_signs;
      o.rht_block = l->rht->block;
      o.rht_scale = (float)(1.0 / std::sqrt((double)l->rht->block));
      o.job0 = jobs;
      o.njobs = pre ? 0 : batch * (l->d_in / l->rht->block);
      jobs += o.njobs;
      if (o.njobs) scratch = std::max(scratch, l->rht->block * 4);
      o.ready = m->d_flags + (size_t)kFlagStride * i;
      o.y = ys[i];
      o.ws = m->d_ws[i];
      o.counters = m->d_cnt[i];
    }
    if (peers) {
      p.n_peers = peers->world;
      p.peer_rank = peers->rank;
      for (int k = 0; k < peers->world; ++k) {
        p.peer_base[k] = static_cast<char*>(peers->y[k]);   // layer 0's y_full on rank k
        p.peer_flag[k] = peers->flag[k];
      }
    }
    p.total_jobs = jobs;
    p.rot_scratch_bytes = scratch;
    p.late_stages = eng_late_stages();
    p.independent = (flags & QP_INDEPENDENT) ? 1 : 0;
    const int grid = (int)std::min<long long>(std::min(num_sms(), kMaxEngCtas), tiles);
    // CTA ranges over the flat tile order, equal in estimated cost: a tile of layer l costs
    // w_l = 1 + E / KT_l (a row tile's epilogue / activation switch, in tiles) + H [half-TCQ: two
    // width runs per row tile]; the CTAs that run rotation jobs take job_tiles fewer tiles per job
    const uint32_t S = tiles;
    const double jt = eng_job_tiles(batch) / rp;
    double wl[kMaxEngOps], cum[kMaxEngOps + 1];
    cum[0] = 0;
    for (int k = 0; k < gr.n; ++k) {
      const EngOp& o = p.op[k];
      wl[k] = 1.0 + eng_row_cost() / o.KT + (o.c_lo != o.c_hi ? eng_half_cost() : 0.0);
      cum[k + 1] = cum[k] + wl[k] * (double)((o.RT / rp) * o.KT);
    }
    auto tile_at = [&](double x) -> double {   // the flat unit index at cumulative cost x
      int k = 0;
      while (k + 1 < gr.n && x >= cum[k + 1]) ++k;
      return p.op[k].tile0 + (x - cum[k]) / wl[k];
    };
    const double base = (cum[gr.n] + jt * jobs) / grid;
    double acc = 0;
    p.cta_begin[0] = 0;
    for (int c = 0; c < grid; ++c) {
      const int my_jobs = c < jobs ? (jobs - 1 - c) / grid + 1 : 0;
      acc += std::max(0.0, base - jt * my_jobs);
      p.cta_begin[c + 1] = (uint32_t)std::min<double>(S, std::llround(tile_at(std::min(acc, cum[gr.n]))));
      if (p.cta_begin[c + 1] < p.cta_begin[c]) p.cta_begin[c + 1] = p.cta_begin[c];
    }
    p.cta_begin[grid] = S;
    cudaError_t e = gr.launch(p, grid, pdl, s);
    if (e != cudaSuccess) return cuda_fail(e, "engine launch");
    count_launch();
  }
  return QP_OK;
}
}  // namespace

// Row-sharded multi-layer forward with the all-gather fused into the engine epilogue: every final y
// value of this rank's rows is stored straight into every rank's y_full over NVLink (peer-mapped
// pointers); the round protocol (entry announcement, per-warp entry gate before the first peer store,
// delivery, wait for every rank's delivery) runs inside each engine launch -- no collective kernel,
// no gather scratch, no permutation (the stores land in the [B][P m] layout), no extra kernels, so
// consecutive launches keep their PDL overlap. The y_full reuse rule of qp_linear_fwd_sharded_p2p holds.
extern "C" qp_status qp_multi_fwd_sharded_p2p(qp_multi* m, const void* const* xs, qp_dtype xt, int batch,
                                              void* const* ys_peers, unsigned* const* flag_peers, int rank,
                                              int world, qp_dtype yt, unsigned flags, void* stream) {
  if (!m || !xs || !ys_peers || !flag_peers)
    return fail(QP_ERR_INVALID_ARG, "NULL argument to qp_multi_fwd_sharded_p2p");
  if (world < 1 || world > kMaxGroup || rank < 0 || rank >= world)
    return fail(QP_ERR_INVALID_ARG, "rank %d / world %d (1..%d ranks)", rank, world, kMaxGroup);
  const int n = (int)m->layers.size();
  for (int k = 0; k < world; ++k)
    if (!flag_peers[k]) return fail(QP_ERR_INVALID_ARG, "flag_peers[%d] is NULL", k);
  for (int i = 0; i < n * world; ++i)
    if (!ys_peers[i]) return fail(QP_ERR_INVALID_ARG, "ys_peers[%d] is NULL", i);
  // every rank's y_full buffers must sit at the same offsets from that rank's layer-0 buffer (the
  // kernel addresses rank k's copy as base_k + offset)
  for (int i = 1; i < n; ++i) {
    const std::ptrdiff_t off = static_cast<const char*>(ys_peers[(size_t)i * world + rank]) -
                               static_cast<const char*>(ys_peers[rank]);
    for (int k = 0; k < world; ++k)
      if (static_cast<const char*>(ys_peers[(size_t)i * world + k]) - static_cast<const char*>(ys_peers[k]) != off)
        return fail(QP_ERR_INVALID_ARG, "qp_multi_fwd_sharded_p2p: layer %d's y_full on rank %d is not at the same "
                    "offset from layer 0's as on this rank. Remedy: carve every rank's y_full buffers out of one "
                    "allocation in the same order (MultiPeerGather does)", i, k);
  }
  if (flags & (QP_Y_ACCUMULATE | QP_INDEPENDENT))
    return fail(QP_ERR_INVALID_ARG, "qp_multi_fwd_sharded_p2p: QP_Y_ACCUMULATE / QP_INDEPENDENT not supported (the "
                "all-gather overwrites y_full; rounds are ordered by the entry barrier)");
  int launches = 0;
  for (const auto& gr : m->groups) {
    if (!gr.launch)
      return fail(QP_ERR_UNSUPPORTED, "qp_multi_fwd_sharded_p2p: layer %d has no engine variant. Remedy: "
                  "qp_linear_fwd_sharded_p2p per layer", gr.first);
    ++launches;
  }
  // (each engine launch is one round: its entry announcement, the per-warp entry gate before the first
  // peer store, the delivery and the wait for every rank's delivery all run inside the engine kernel)
  (void)launches;
  const EngPeers pe{world, rank, ys_peers, flag_peers};
  // ys: this rank's own y_full (argument checks only; the engine stores through pe)
  std::vector<void*> own(n);
  for (int i = 0; i < n; ++i) own[i] = ys_peers[(size_t)i * world + rank];
  return multi_fwd_impl(m, xs, xt, batch, own.data(), yt, flags, stream, &pe);
}

// Row-sharded multi-layer forward: the engine over this rank's shards (one persistent launch per
// table family) into each shard's local scratch, then ONE grouped NCCL all-gather of every layer's
// rows (ncclGroupStart / End: a single collective launch over NVLink / NVSwitch), then the
// [P][B][m] -> [B][P m] permutation for batch > 1.
extern "C" qp_status qp_multi_fwd_sharded(qp_multi* m, const void* const* xs, qp_dtype xt, int batch,
                                          void* const* ys_full, qp_dtype yt, void* comm, unsigned flags,
                                          void* stream) {
  if (!m || !xs || !ys_full || !comm) return fail(QP_ERR_INVALID_ARG, "NULL argument to qp_multi_fwd_sharded");
  if (flags & QP_Y_ACCUMULATE)
    return fail(QP_ERR_INVALID_ARG, "qp_multi_fwd_sharded: QP_Y_ACCUMULATE is not supported (the all-gather "
                "overwrites y_full)");
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  int world = 0;
  if (ncclCommCount(c, &world) != ncclSuccess || world < 1) return fail(QP_ERR_NCCL, "ncclCommCount failed");
  const int n = (int)m->layers.size();
  const int eb = yt == QP_F32 ? 4 : 2;
  std::vector<void*> local(n);
  for (int i = 0; i < n; ++i) {
    const qp_layer* l = m->layers[i];
    if (!ys_full[i]) return fail(QP_ERR_INVALID_ARG, "ys_full[%d] is NULL", i);
    if (l->gather_bytes < (size_t)(world + 1) * batch * l->d_out * eb)
      return fail(QP_ERR_CONFIG_MISMATCH, "qp_multi_fwd_sharded: layer %d is not a shard of a %d-rank split "
                  "(qp_layer_shard)", i, world);
    local[i] = l->d_gather;
  }
  // (QP_INDEPENDENT is dropped: the next engine launch must not overwrite the local rows while the
  // preceding all-gather still reads them)
  qp_status st = qp_multi_fwd(m, xs, xt, batch, local.data(), yt, flags & ~QP_INDEPENDENT, stream);
  if (st != QP_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ncclResult_t r = ncclGroupStart();
  for (int i = 0; i < n && r == ncclSuccess; ++i) {
    const qp_layer* l = m->layers[i];
    uint8_t* gathered = static_cast<uint8_t*>(l->d_gather) + (size_t)batch * l->d_out * eb;
    r = ncclAllGather(local[i], batch == 1 ? ys_full[i] : gathered, (size_t)batch * l->d_out,
                      yt == QP_F32 ? ncclFloat32 : ncclFloat16, c, s);
  }
  ncclResult_t r2 = ncclGroupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess)
    return fail(QP_ERR_NCCL, "grouped ncclAllGather: %s", ncclGetErrorString(r != ncclSuccess ? r : r2));
  if (batch > 1) {
    for (int i = 0; i < n; ++i) {
      const qp_layer* l = m->layers[i];
      uint8_t* gathered = static_cast<uint8_t*>(l->d_gather) + (size_t)batch * l->d_out * eb;
      cudaError_t e = launch_gather_permute(gathered, ys_full[i], world, batch, l->d_out, eb, s);
      if (e != cudaSuccess) return cuda_fail(e, "gather permute");
    }
  }
  // asynchronous NCCL faults of earlier collectives surface here (header contract)
  ncclResult_t ae = ncclSuccess;
  if (ncclCommGetAsyncError(c, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress)
    return fail(QP_ERR_NCCL, "asynchronous NCCL error: %s", ncclGetErrorString(ae));
  return QP_OK;
}

// ---------------------------------------------------------------------------------------
// K (column) sharding: row-parallel layers (the down projection after a column-parallel up /
// gate): rank r owns input columns [r*d_in/world, (r+1)*d_in/world) of every row and computes a
// partial y over all rows; the partials are summed across ranks (ncclAllReduce).
// ---------------------------------------------------------------------------------------
extern "C" qp_status qp_layer_shard_k(const qp_layer* l, int rank, int world, qp_layer** out) {
  if (!l || !out) return fail(QP_ERR_INVALID_ARG, "NULL argument to qp_layer_shard_k");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return fail(QP_ERR_INVALID_ARG, "rank %d / world %d", rank, world);
  if (l->c_lo != l->c_hi)
    return fail(QP_ERR_UNSUPPORTED, "qp_layer_shard_k: half-TCQ layers (two widths along d_in) are not column-"
                "sharded. Remedy: row-shard them (qp_layer_shard) or use a single-width quantizer");
  const qp_rht* pr = l->rht;
  if (l->d_in % world)
    return fail(QP_ERR_PARTITION_MISMATCH, "d_in=%d does not split into %d column blocks", l->d_in, world);
  const int dl = l->d_in / world;
  if (dl % kTileCols || dl % pr->block)
    return fail(QP_ERR_PARTITION_MISMATCH, "column block %d must be a multiple of 256 (k tiles) and of the rotation "
                "block %d (R is block-diagonal: a shard rotates only its own blocks). Remedy: quantize with a "
                "smaller rotation block (qp_rht_create(seed, d_in, block))", dl, pr->block);
  // the rotation of the shard = the blocks of its columns: same block size, the sign slice
  auto r = new qp_rht();
  r->seed = pr->seed;
  r->d_in = dl;
  r->block = pr->block;
  r->sign_bits.assign((dl + 31) / 32, 0u);
  const int c0 = rank * dl;
  for (int i = 0; i < dl; ++i)
    if ((pr->sign_bits[(c0 + i) >> 5] >> ((c0 + i) & 31)) & 1u) r->sign_bits[i >> 5] |= 1u << (i & 31);
  r->d_signs = static_cast<uint32_t*>(dev_alloc(r->sign_bits.size() * 4));
  if (!r->d_signs || cudaMemcpy(r->d_signs, r->sign_bits.data(), r->sign_bits.size() * 4, cudaMemcpyHostToDevice) !=
                         cudaSuccess) {
    dev_free(r->d_signs);
    delete r;
    return fail(QP_ERR_ALLOC, "shard rotation allocation failed");
  }
  auto s = new qp_layer();
  s->owned_rht = r;
  qp_status st = layer_init(s, l->d_out, dl, l->scheme, l->bits_x4, l->cb, r);
  if (st != QP_OK) {
    layer_release(s);
    delete s;
    return st;
  }
  // every row tile's k tiles [kt0, kt0 + KTl): one strided copy (row-tile-major storage)
  const size_t tile = 512 * (size_t)l->c_lo, KT = l->d_in / kTileCols, KTl = dl / kTileCols;
  const size_t RT = l->d_out / kTileRows;
  cudaError_t e = cudaMemcpy2D(s->d_codes, KTl * tile, l->d_codes + (size_t)rank * KTl * tile, KT * tile, KTl * tile,
                               RT, cudaMemcpyDeviceToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(s->d_scales, l->d_scales, (size_t)l->d_out * 4, cudaMemcpyDeviceToDevice);
  if (e == cudaSuccess) e = cudaStreamSynchronize(0);
  if (e != cudaSuccess) {
    layer_release(s);
    delete s;
    return cuda_fail(e, "k-shard copy");
  }
  *out = s;
  return QP_OK;
}

extern "C" qp_status qp_linear_fwd_ksharded(const qp_layer* shard, const void* x_local, qp_dtype xt, int batch, void* y,
                                            qp_dtype yt, void* comm, unsigned flags, void* stream) {
  if (!shard || !y || !comm) return fail(QP_ERR_INVALID_ARG, "NULL argument to qp_linear_fwd_ksharded");
  if (yt != QP_F32) return fail(QP_ERR_INVALID_ARG, "qp_linear_fwd_ksharded: partial sums need fp32 y");
  if (flags & QP_Y_ACCUMULATE)
    return fail(QP_ERR_INVALID_ARG, "qp_linear_fwd_ksharded: QP_Y_ACCUMULATE would be summed world times. "
                "Remedy: add the residual after the call");
  qp_status st = qp_linear_fwd(shard, x_local, xt, batch, y, yt, flags, stream);
  if (st != QP_OK) return st;
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  ncclResult_t r = ncclAllReduce(y, y, (size_t)batch * shard->d_out, ncclFloat32, ncclSum, c,
                                 static_cast<cudaStream_t>(stream));
  if (r != ncclSuccess) return fail(QP_ERR_NCCL, "ncclAllReduce: %s", ncclGetErrorString(r));
  ncclResult_t ae = ncclSuccess;
  if (ncclCommGetAsyncError(c, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress)
    return fail(QP_ERR_NCCL, "asynchronous NCCL error: %s", ncclGetErrorString(ae));
  return QP_OK;
}
