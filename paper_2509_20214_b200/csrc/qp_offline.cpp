// Data-free offline quantization (host, multithreaded): qp_quantize_offline.
//
//   W' = W R^T (each row rotated), s_j = RMS(W'_j) (reading R10), W~ = W' / s,
//   then per LAYOUT.md unit (one lane of one tile = 128 weight pairs):
//     NUQ / UNIF  RTN per scalar: argmin |v - LUT[i]|, lowest index on ties
//     VQ          RTN per pair:   argmin ||v - LUT[i]||^2
//     TCQ         tail-biting Viterbi, rotate-half (reading R4)
//   and the codes are packed MSB-first into the lane's word stream.
// Arithmetic is double precision so that, given the same W~, the decisions match the
// NumPy oracle (ties: lowest index / lowest predecessor, reading R5).
#include <cuda_fp16.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

#include "../../include/qpalette.h"
#include "qp_internal.h"

namespace {

float h2f(uint16_t b) {
  __half h;
  std::memcpy(&h, &b, 2);
  return __half2float(h);
}

uint64_t splitmix64(uint64_t seed, uint64_t i) {
  uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// In-place fast Walsh-Hadamard transform (natural/Sylvester order) of one block.
void fwht(double* v, int n) {
  for (int h = 1; h < n; h <<= 1)
    for (int i = 0; i < n; i += 2 * h)
      for (int j = i; j < i + h; ++j) {
        const double a = v[j], b = v[j + h];
        v[j] = a + b;
        v[j + h] = a - b;
      }
}

// step j of lane l -> (row, col) in the 32 x 256 tile (LAYOUT.md)
inline void step_pos(int lane, int j, int* row, int* col) {
  const int g = lane >> 2, q = lane & 3, kap = j >> 3, m = (j >> 2) & 1, rho = j & 3;
  *row = 16 * m + g + 8 * (rho & 1);
  *col = 64 * q + 4 * kap + 2 * (rho >> 1);
}

struct Viterbi {
  int L, s, n;
  const std::vector<double>* lut;   // [2^L][2]
  std::vector<double> D, Dn;
  std::vector<uint16_t> bp;         // [n][2^(L-s)]
  Viterbi(int L_, int s_, int n_, const std::vector<double>* lut_) : L(L_), s(s_), n(n_), lut(lut_) {
    const int ns = 1 << (L >= s ? L - s : 0);
    D.resize(ns);
    Dn.resize(ns);
    bp.resize((size_t)n * ns);
  }
  // start < 0: free start; end < 0: free end (argmin, lowest index). Returns cost, fills windows.
  double run(const double* v, int start, int end, uint32_t* windows) {
    const int ns = 1 << (L - s), nk = 1 << s;
    const double inf = std::numeric_limits<double>::infinity();
    for (int i = 0; i < ns; ++i) D[i] = (start < 0 || i == start) ? 0.0 : inf;
    const double* T = lut->data();
    for (int i = 0; i < n; ++i) {
      const double v0 = v[2 * i], v1 = v[2 * i + 1];
      uint16_t* bpi = bp.data() + (size_t)i * ns;
      for (int sp = 0; sp < ns; ++sp) {
        double best = inf;
        int bk = 0;
        for (int k = 0; k < nk; ++k) {
          const int w = k * ns + sp;
          const double d0 = v0 - T[2 * w], d1 = v1 - T[2 * w + 1];
          const double c = D[w >> s] + (d0 * d0 + d1 * d1);
          if (c < best) {
            best = c;
            bk = k;
          }
        }
        Dn[sp] = best;
        bpi[sp] = (uint16_t)bk;
      }
      std::swap(D, Dn);
    }
    int sig = end;
    if (sig < 0) {
      sig = 0;
      for (int i = 1; i < ns; ++i)
        if (D[i] < D[sig]) sig = i;
    }
    const double cost = D[sig];
    for (int i = n - 1; i >= 0; --i) {
      const int k = bp[(size_t)i * ns + sig];
      const uint32_t w = (uint32_t)(k * ns + sig);
      windows[i] = w;
      sig = (int)(w >> s);
    }
    return cost;
  }
};

// rotate-half tail-biting encoder (reading R4)
void tcq_encode(Viterbi& vit, const double* v, uint32_t* windows) {
  const int n = vit.n, h = n / 2, L = vit.L, s = vit.s;
  std::vector<double> rolled(2 * n);
  for (int i = 0; i < n; ++i) {
    const int src = (i + h) % n;
    rolled[2 * i] = v[2 * src];
    rolled[2 * i + 1] = v[2 * src + 1];
  }
  std::vector<uint32_t> wr(n);
  vit.run(rolled.data(), -1, -1, wr.data());
  const int S = (int)(wr[n - h - 1] & ((1u << (L - s)) - 1u));
  vit.run(v, S, S, windows);
}

void put_bits(std::vector<uint32_t>& words, int pos, uint32_t value, int nbits) {
  for (int b = 0; b < nbits; ++b) {
    const uint32_t bit = (value >> (nbits - 1 - b)) & 1u;
    const int t = pos + b;
    words[t >> 5] |= bit << (31 - (t & 31));
  }
}

}  // namespace

extern "C" qp_status qp_quantize_offline(const float* W_host, int d_out, int d_in, qp_scheme scheme, int bits_x4,
                                         const qp_codebook* cb, const qp_rht* r, int n_threads, qp_layer** out);

namespace qp {
size_t tcq_viterbi_scratch_bytes(int L, int s, int grid);
cudaError_t launch_tcq_viterbi(const double* v, int units, int L, int s, int tb, const double* tlut_dev,
                               uint32_t* windows, uint16_t* bp_scratch, int grid, cudaStream_t st);
}

namespace {
// Rotate-half Viterbi of every TCQ unit with k-tile class c on the GPU (qp_encode.cu): fills
// win_all[u * 128 ..] for the units in `ids`. Bitwise the host encoder's windows.
qp_status gpu_tcq_windows(const std::vector<double>& v_all, const std::vector<long long>& ids, int L, int s, int tb,
                          const uint16_t* host_tlut, std::vector<uint32_t>& win_all) {
  if (ids.empty()) return QP_OK;
  const size_t nu = ids.size();
  std::vector<double> v(nu * 256);
  for (size_t i = 0; i < nu; ++i) std::memcpy(&v[i * 256], &v_all[(size_t)ids[i] * 256], 256 * sizeof(double));
  std::vector<double> tl((size_t)2 << tb);
  for (size_t i = 0; i < tl.size(); ++i) tl[i] = h2f(host_tlut[i]);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::min<size_t>((size_t)sms, nu);
  double *d_v = nullptr, *d_tl = nullptr;
  uint32_t* d_w = nullptr;
  uint16_t* d_bp = nullptr;
  cudaError_t e = cudaMalloc(&d_v, v.size() * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_tl, tl.size() * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&d_w, nu * 128 * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMalloc(&d_bp, qp::tcq_viterbi_scratch_bytes(L, s, grid));
  if (e == cudaSuccess) e = cudaMemcpy(d_v, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d_tl, tl.data(), tl.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = qp::launch_tcq_viterbi(d_v, (int)nu, L, s, tb, d_tl, d_w, d_bp, grid, nullptr);
  std::vector<uint32_t> w(nu * 128);
  if (e == cudaSuccess) e = cudaMemcpy(w.data(), d_w, w.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost);
  cudaFree(d_v);
  cudaFree(d_tl);
  cudaFree(d_w);
  cudaFree(d_bp);
  if (e != cudaSuccess) return (qp_status)qp::set_error(QP_ERR_CUDA, cudaGetErrorString(e));
  for (size_t i = 0; i < nu; ++i) std::memcpy(&win_all[(size_t)ids[i] * 128], &w[i * 128], 128 * sizeof(uint32_t));
  return QP_OK;
}
}  // namespace

static qp_status quantize_offline_impl(const float* W_host, int d_out, int d_in, qp_scheme scheme, int bits_x4,
                                       const qp_codebook* cb, const qp_rht* r, int n_threads, bool gpu,
                                       qp_layer** out);

qp_status qp_quantize_offline(const float* W_host, int d_out, int d_in, qp_scheme scheme, int bits_x4,
                              const qp_codebook* cb, const qp_rht* r, int n_threads, qp_layer** out) {
  return quantize_offline_impl(W_host, d_out, d_in, scheme, bits_x4, cb, r, n_threads, false, out);
}

extern "C" qp_status qp_quantize_offline_gpu(const float* W_host, int d_out, int d_in, qp_scheme scheme,
                                             int bits_x4, const qp_codebook* cb, const qp_rht* r, int n_threads,
                                             qp_layer** out) {
  return quantize_offline_impl(W_host, d_out, d_in, scheme, bits_x4, cb, r, n_threads, true, out);
}

// accessors implemented in qp_host.cpp (objects are opaque here)
extern "C" {
qp_status qp_internal_codebook_info(const qp_codebook* cb, int* L, int* tb, const uint16_t** host, size_t* n);
qp_status qp_internal_rht_info(const qp_rht* r, uint64_t* seed, int* d_in, int* block, const uint32_t** sign_bits);
qp_status qp_internal_codebook_alpha(const qp_codebook* cb, double* alpha);
}

static qp_status quantize_offline_impl(const float* W_host, int d_out, int d_in, qp_scheme scheme, int bits_x4,
                                       const qp_codebook* cb, const qp_rht* r, int n_threads, bool gpu,
                                       qp_layer** out) {
  if (!W_host || !cb || !r || !out) return QP_ERR_INVALID_ARG;
  *out = nullptr;
  int L = 0, tb = 0, rd_in = 0, block = 0;
  const uint16_t* host = nullptr;
  size_t nh = 0;
  uint64_t seed = 0;
  const uint32_t* sign_bits = nullptr;
  qp_status st = qp_internal_codebook_info(cb, &L, &tb, &host, &nh);
  if (st != QP_OK) return st;
  if ((st = qp_internal_rht_info(r, &seed, &rd_in, &block, &sign_bits)) != QP_OK) return st;
  double alpha = 1.0;   // reconstruction scale (reading R22): W~ = W' / (s alpha), stored scale s alpha
  if ((st = qp_internal_codebook_alpha(cb, &alpha)) != QP_OK) return st;
  if (rd_in != d_in) return QP_ERR_CONFIG_MISMATCH;
  if (d_out <= 0 || d_in <= 0 || d_out % 32 || d_in % 256) return QP_ERR_PARTITION_MISMATCH;
  if (n_threads <= 0) n_threads = (int)std::max(1u, std::thread::hardware_concurrency());

  // ---- 1. rotate rows, per-output-channel RMS scales ----------------------------
  std::vector<double> Wt((size_t)d_out * d_in);
  std::vector<float> scales(d_out);
  const double inv = 1.0 / std::sqrt((double)block);
  auto rotate_rows = [&](int r0, int r1) {
    for (int j = r0; j < r1; ++j) {
      double* row = Wt.data() + (size_t)j * d_in;
      for (int i = 0; i < d_in; ++i) {
        const double sgn = (sign_bits[i >> 5] >> (i & 31)) & 1u ? -1.0 : 1.0;
        row[i] = sgn * (double)W_host[(size_t)j * d_in + i];
      }
      for (int o = 0; o < d_in; o += block) fwht(row + o, block);
      double ss = 0;
      for (int i = 0; i < d_in; ++i) {
        row[i] *= inv;
        ss += row[i] * row[i];
      }
      double sc = std::sqrt(ss / d_in) * alpha;
      scales[j] = (float)sc;
      const double is = sc > 0 ? 1.0 / sc : 0.0;
      for (int i = 0; i < d_in; ++i) row[i] *= is;
    }
  };
  {
    std::vector<std::thread> th;
    const int per = (d_out + n_threads - 1) / n_threads;
    for (int t = 0; t < n_threads; ++t) {
      const int a = t * per, b = std::min(d_out, a + per);
      if (a < b) th.emplace_back(rotate_rows, a, b);
    }
    for (auto& x : th) x.join();
  }

  // ---- 2. codebook in double -------------------------------------------------------------
  const bool tcq = scheme == QP_TCQ || scheme == QP_HALF_TCQ;
  std::vector<double> lut;   // TCQ: [2^L][2]; VQ: [2^c][2]; NUQ/UNIF: [2^b]
  if (tcq) {
    // hybrid LUT quantlut_sym(tlut, L, tb) (generalised for L != 16: reading R1)
    lut.resize((size_t)2 << L);
    for (uint32_t w = 0; w < (1u << L); ++w) {
      const uint32_t p = (uint32_t)(((uint64_t)(w + 1) * w) & ((1ull << L) - 1));
      const bool neg = (p >> (L - 1)) & 1u;
      const uint32_t idx = (p >> (L - tb - 1)) & ((1u << tb) - 1u);
      const double t0 = h2f(host[2 * idx]), t1 = h2f(host[2 * idx + 1]);
      lut[2 * w] = neg ? -t0 : t0;
      lut[2 * w + 1] = t1;
    }
  } else {
    lut.resize(nh);
    for (size_t i = 0; i < nh; ++i) lut[i] = h2f(host[i]);
  }

  // ---- 3. encode every (tile, lane) unit ---------------------------------------------------
  int c_lo, c_hi;
  if (scheme == QP_HALF_TCQ) {
    c_lo = (bits_x4 - 1) / 2;
    c_hi = c_lo + 1;
  } else {
    c_lo = c_hi = bits_x4 / 2;
  }
  const int RT = d_out / 32, KT = d_in / 256, KH = KT / 2;
  const size_t rowtile_bytes = (size_t)KH * 512 * c_lo + (size_t)(KT - KH) * 512 * c_hi;
  std::vector<uint8_t> codes(rowtile_bytes * RT, 0);
  const long long units = (long long)RT * KT * 32;
  // the trellis input of unit u (tile u / 32, lane u % 32): 128 weight pairs in step order
  auto gather = [&](long long u, double* v) {
    const int lane = (int)(u % 32);
    const long long tile = u / 32;
    const int rt = (int)(tile / KT), kt = (int)(tile % KT);
    for (int j = 0; j < 128; ++j) {
      int row, col;
      step_pos(lane, j, &row, &col);
      const double* src = Wt.data() + (size_t)(rt * 32 + row) * d_in + kt * 256 + col;
      v[2 * j] = src[0];
      v[2 * j + 1] = src[1];
    }
  };
  std::vector<uint32_t> gpu_win;   // GPU-encoded windows of every TCQ unit [units][128]
  if (tcq && gpu) {
    std::vector<double> v_all((size_t)units * 256);
    for (long long u = 0; u < units; ++u) gather(u, &v_all[(size_t)u * 256]);
    gpu_win.resize((size_t)units * 128);
    std::vector<long long> lo, hi;
    for (long long u = 0; u < units; ++u) (((u / 32) % KT) < KH ? lo : hi).push_back(u);
    if (c_lo == c_hi) {
      lo.insert(lo.end(), hi.begin(), hi.end());
      hi.clear();
      std::sort(lo.begin(), lo.end());
    }
    if ((st = gpu_tcq_windows(v_all, lo, L, c_lo, tb, host, gpu_win)) != QP_OK) return st;
    if ((st = gpu_tcq_windows(v_all, hi, L, c_hi, tb, host, gpu_win)) != QP_OK) return st;
  }
  std::atomic<long long> next{0};
  auto worker = [&]() {
    std::vector<double> v(256);
    std::vector<uint32_t> win(128);
    // trellis state only for TCQ (L = 0 for the other schemes)
    Viterbi vlo(tcq ? L : c_lo, c_lo, 128, &lut), vhi(tcq ? L : c_hi, c_hi, 128, &lut);
    for (;;) {
      const long long u = next.fetch_add(1);
      if (u >= units) break;
      const int lane = (int)(u % 32);
      const long long tile = u / 32;
      const int rt = (int)(tile / KT), kt = (int)(tile % KT);
      const int c = (kt < KH) ? c_lo : c_hi;
      for (int j = 0; j < 128; ++j) {
        int row, col;
        step_pos(lane, j, &row, &col);
        const double* src = Wt.data() + (size_t)(rt * 32 + row) * d_in + kt * 256 + col;
        v[2 * j] = src[0];
        v[2 * j + 1] = src[1];
      }
      std::vector<uint32_t> words(4 * c, 0u);
      if (tcq) {
        if (gpu)
          std::memcpy(win.data(), &gpu_win[(size_t)u * 128], 128 * sizeof(uint32_t));
        else
          tcq_encode(kt < KH ? vlo : vhi, v.data(), win.data());
        for (int j = 0; j < 128; ++j) put_bits(words, j * c, win[j] >> (L - c), c);   // top s bits of w_j
      } else if (scheme == QP_VQ) {
        const int ne = 1 << c;
        for (int j = 0; j < 128; ++j) {
          int best = 0;
          double bd = std::numeric_limits<double>::infinity();
          for (int e = 0; e < ne; ++e) {
            const double d0 = v[2 * j] - lut[2 * e], d1 = v[2 * j + 1] - lut[2 * e + 1];
            const double d = d0 * d0 + d1 * d1;
            if (d < bd) {
              bd = d;
              best = e;
            }
          }
          put_bits(words, j * c, (uint32_t)best, c);
        }
      } else {
        const int b = c / 2, ne = 1 << b;
        for (int j = 0; j < 128; ++j) {
          uint32_t idx2[2];
          for (int h = 0; h < 2; ++h) {
            int best = 0;
            double bd = std::numeric_limits<double>::infinity();
            for (int e = 0; e < ne; ++e) {
              const double d = std::fabs(v[2 * j + h] - lut[e]);
              if (d < bd) {
                bd = d;
                best = e;
              }
            }
            idx2[h] = (uint32_t)best;
          }
          put_bits(words, j * c, (idx2[0] << b) | idx2[1], c);
        }
      }
      const size_t base = (size_t)rt * rowtile_bytes +
                          (kt < KH ? (size_t)kt * 512 * c_lo : (size_t)KH * 512 * c_lo + (size_t)(kt - KH) * 512 * c_hi);
      for (int i = 0; i < 4 * c; ++i) {
        const size_t off = base + ((size_t)(i / 4) * 32 + lane) * 16 + (i % 4) * 4;
        std::memcpy(codes.data() + off, &words[i], 4);   // little-endian host
      }
    }
  };
  {
    std::vector<std::thread> th;
    for (int t = 0; t < n_threads; ++t) th.emplace_back(worker);
    for (auto& x : th) x.join();
  }
  return qp_layer_from_codes(codes.data(), codes.size(), scales.data(), d_out, d_in, scheme, bits_x4, cb, r, out);
}
