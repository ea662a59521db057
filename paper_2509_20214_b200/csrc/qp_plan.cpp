// Host-only planning helpers of the C ABI (no device work).
//
// qp_optimal_bits: Theorem 1 of the paper, optimal fractional bit allocation with
// ideal Gaussian quantizers, b_l* = max{eta, ln(a_l / n_l) / (2 ln 2) + C} with the C that makes
// the memory budget tight. S(C) = sum_l max{eta, u_l + C} n_l is piecewise linear and
// non-decreasing in C with breakpoints C_l = eta - u_l; the exact C is found by sorting the
// breakpoints and solving the linear piece on which S crosses M (no iteration).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <numeric>
#include <string>
#include <vector>

#include "qpalette.h"
#include "qp_internal.h"

namespace {
qp_status fail(qp_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  return (qp_status)qp::set_error((int)s, buf);
}
}  // namespace

extern "C" qp_status qp_optimal_bits(const double* a, const double* n, int L, double M, double eta, double* b_out) {
  if (!a || !n || !b_out || L <= 0) return fail(QP_ERR_INVALID_ARG, "qp_optimal_bits: NULL argument or L <= 0");
  double total = 0.0;
  std::vector<double> u(L);
  for (int l = 0; l < L; ++l) {
    if (!(a[l] > 0.0) || !(n[l] > 0.0) || !std::isfinite(a[l]) || !std::isfinite(n[l]))
      return fail(QP_ERR_INVALID_ARG, "qp_optimal_bits: a[%d]=%g, n[%d]=%g must be positive and finite", l, a[l], l,
                      n[l]);
    u[l] = std::log(a[l] / n[l]) / (2.0 * std::log(2.0));
    total += n[l];
  }
  if (!(eta >= 0.0) || !std::isfinite(M))
    return fail(QP_ERR_INVALID_ARG, "qp_optimal_bits: eta=%g must be >= 0 and M finite", eta);
  if (M < eta * total * (1.0 - 1e-12))
    return fail(QP_ERR_CONFIG_MISMATCH, "qp_optimal_bits: budget M=%g below eta * sum(n) = %g (P:172)", M,
                    eta * total);
  // layers leave the floor in order of increasing breakpoint eta - u_l (decreasing u_l)
  std::vector<int> ord(L);
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](int x, int y) { return u[x] > u[y]; });
  // with the first k layers (in that order) free: S(C) = eta * (total - N_k) + sum_{free} (u_l + C) n_l
  double Nk = 0.0, Uk = 0.0, C = 0.0;
  for (int k = 0; k < L; ++k) {
    const int l = ord[k];
    Nk += n[l];
    Uk += u[l] * n[l];
    C = (M - eta * (total - Nk) - Uk) / Nk;            // solve S(C) = M on this piece
    const double next_bp = k + 1 < L ? eta - u[ord[k + 1]] : INFINITY;
    if (C <= next_bp) break;                            // the next layer stays on the floor
  }
  for (int l = 0; l < L; ++l) b_out[l] = std::max(eta, u[l] + C);
  return QP_OK;
}

// ---------------------------------------------------------------------------------------------
// qp_plan_msq: fusion-aware mixed-scheme quantization, exact.
//
// Each block decomposes into four independent choices that share only the budget: the QKV part
// (a partition of {q,k,v} into fusible groups, one quantizer per group), o, the UG part (u and g
// separate or fused) and d. Every choice is an option (loss, cost); the problem is a multiple-
// choice knapsack over 4B classes. Exact solution by Pareto frontiers: the partial solutions after
// each class are pruned to the (cost, loss)-nondominated ones (an optimal solution's prefixes are
// nondominated), then merged with the next class's own frontier. The best frontier point within
// the budget is traced back to the choices.
// ---------------------------------------------------------------------------------------------
namespace {

constexpr int kGroupTypes = 12;   // q, k, v, qk, qv, kv, qkv, o, u, g, ug, d
const int kGroupLayers[kGroupTypes][3] = {{0, -1, -1}, {1, -1, -1}, {2, -1, -1}, {0, 1, -1}, {0, 2, -1}, {1, 2, -1},
                                          {0, 1, 2},   {3, -1, -1}, {4, -1, -1}, {5, -1, -1}, {4, 5, -1}, {6, -1, -1}};

struct Opt {
  double loss, cost;
  int g[3], q[3];   // up to 3 (group type, quantizer) pairs; g = -1 unused
};

// nondominated subset of `v` (sorted by cost ascending, strictly decreasing loss)
template <class T, class Cost, class Loss>
std::vector<T> pareto(std::vector<T> v, Cost cost, Loss loss) {
  std::sort(v.begin(), v.end(), [&](const T& a, const T& b) {
    return cost(a) < cost(b) || (cost(a) == cost(b) && loss(a) < loss(b));
  });
  std::vector<T> out;
  for (const T& x : v)
    if (out.empty() || loss(x) < loss(out.back())) out.push_back(x);
  return out;
}

}  // namespace

extern "C" qp_status qp_plan_msq(int n_blocks, const double* a, int n_quant, const double* err, const double* cost,
                                 double budget, int fusion, int* group_out, int* quant_out, double* loss_out,
                                 double* cost_out) {
  if (n_blocks <= 0 || n_quant <= 0 || !a || !err || !cost || !group_out || !quant_out)
    return fail(QP_ERR_INVALID_ARG, "qp_plan_msq: NULL argument or empty problem");
  const int nq = n_quant;
  // classes: per block QKV part, o, UG part, d
  auto layer_loss = [&](int b, int l, int q) { return a[b * 7 + l] * err[q]; };
  std::vector<std::vector<Opt>> classes;
  for (int b = 0; b < n_blocks; ++b) {
    // partitions of {q,k,v}: {q}{k}{v}, {qk}{v}, {qv}{k}, {kv}{q}, {qkv}; of {u,g}: {u}{g}, {ug}
    const std::vector<std::vector<int>> qkv_parts = fusion ? std::vector<std::vector<int>>{{0, 1, 2}, {3, 2}, {4, 1}, {5, 0}, {6}}
                                                           : std::vector<std::vector<int>>{{0, 1, 2}};
    const std::vector<std::vector<int>> ug_parts = fusion ? std::vector<std::vector<int>>{{8, 9}, {10}}
                                                          : std::vector<std::vector<int>>{{8, 9}};
    const std::vector<std::vector<std::vector<int>>> sets = {qkv_parts, {{7}}, ug_parts, {{11}}};
    for (const auto& parts : sets) {
      std::vector<Opt> opts;
      for (const auto& part : parts) {
        const int ng = (int)part.size();
        int total = 1;
        for (int i = 0; i < ng; ++i) total *= nq;
        for (int code = 0; code < total; ++code) {
          Opt o{};
          o.loss = 0;
          o.cost = 0;
          int c = code;
          for (int i = 0; i < 3; ++i) o.g[i] = -1;
          for (int i = 0; i < ng; ++i) {
            const int q = c % nq;
            c /= nq;
            const int g = part[i];
            o.g[i] = g;
            o.q[i] = q;
            o.cost += cost[g * nq + q];
            for (int j = 0; j < 3 && kGroupLayers[g][j] >= 0; ++j) o.loss += layer_loss(b, kGroupLayers[g][j], q);
          }
          opts.push_back(o);
        }
      }
      classes.push_back(pareto(opts, [](const Opt& o) { return o.cost; }, [](const Opt& o) { return o.loss; }));
    }
  }
  // frontier merge with back pointers
  struct Node {
    double loss, cost;
    int prev, opt;
  };
  std::vector<std::vector<Node>> fronts;
  std::vector<Node> cur = {{0.0, 0.0, -1, -1}};
  const size_t kMaxFront = 4000000;
  for (size_t c = 0; c < classes.size(); ++c) {
    std::vector<Node> next;
    next.reserve(cur.size() * classes[c].size());
    for (int i = 0; i < (int)cur.size(); ++i)
      for (int j = 0; j < (int)classes[c].size(); ++j) {
        const double nc = cur[i].cost + classes[c][j].cost;
        if (nc > budget * (1 + 1e-12)) continue;
        next.push_back({cur[i].loss + classes[c][j].loss, nc, i, j});
      }
    if (next.empty()) return fail(QP_ERR_CONFIG_MISMATCH, "qp_plan_msq: budget %g below the cheapest assignment", budget);
    next = pareto(next, [](const Node& n) { return n.cost; }, [](const Node& n) { return n.loss; });
    if (next.size() > kMaxFront) return fail(QP_ERR_ALLOC, "qp_plan_msq: Pareto frontier exceeds %zu points", kMaxFront);
    fronts.push_back(cur);
    cur.swap(next);
  }
  // best within budget: the frontier is sorted by cost with decreasing loss -> the last point
  int idx = (int)cur.size() - 1;
  if (loss_out) *loss_out = cur[idx].loss;
  if (cost_out) *cost_out = cur[idx].cost;
  for (int c = (int)classes.size() - 1; c >= 0; --c) {
    const Node& n = (c == (int)classes.size() - 1) ? cur[idx] : fronts[c + 1][idx];
    const Opt& o = classes[c][n.opt];
    const int b = c / 4;
    for (int i = 0; i < 3 && o.g[i] >= 0; ++i)
      for (int j = 0; j < 3 && kGroupLayers[o.g[i]][j] >= 0; ++j) {
        group_out[b * 7 + kGroupLayers[o.g[i]][j]] = o.g[i];
        quant_out[b * 7 + kGroupLayers[o.g[i]][j]] = o.q[i];
      }
    idx = n.prev;
  }
  return QP_OK;
}
