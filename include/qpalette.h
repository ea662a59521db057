/*
 * qpalette.h -- C ABI of the B200 (sm_100a) Q-Palette hot path.
 *
 * What the library computes (Q-Palette, arXiv 2509.20214; "P:n" = line n of the
 * paper source /root/reference/PAPER.md, "S:n" = line n of SPEC.md):
 *
 *     y[beta] = diag(s) * W_hat * (R x[beta]),   beta = 0 .. batch-1,  batch in 1..8
 *
 *   R      randomized Hadamard rotation of the input dimension only:
 *          R = (1/sqrt(b)) * blockdiag(H_b, ..., H_b) * D, H_b Sylvester, D = diag(+-1)
 *          drawn from splitmix64(seed, i); b = largest power-of-two divisor of d_in.
 *   W_hat  weights decoded on the fly from fractional-bit codes:
 *          TCQ / half-TCQ (bitshift trellis, hybrid `quantlut_sym` codebook, tail-biting),
 *          2-D VQ, NUQ and uniform scalar quantization.
 *   s      per-output-channel scales.
 *
 * Code layout: LAYOUT.md (tiles of 32 rows x 256 columns, row-tile-major, one trellis /
 * code run of 256 weights per lane, MSB-first 32-bit word streams).
 *
 * Conventions (apply to every entry point):
 *   - Ownership: the caller owns x, y, W and every host buffer; the library owns the
 *     device memory of codebooks, rotations, layers and groups (allocated through the
 *     hook of qp_set_allocator if set, else cudaMalloc) and frees it in qp_*_free.
 *     A layer references (does not own) its codebook and rotation: free layers first.
 *   - Asynchrony: argument/shape validation is synchronous and returns a status; all
 *     device work is enqueued on `stream` (a cudaStream_t, passed as void*) with no
 *     implicit synchronisation. Asynchronous CUDA faults surface as QP_ERR_CUDA on a
 *     later call. A layer or group object may be used by one stream at a time (it owns
 *     a small scratch buffer); distinct objects may be used concurrently.
 *   - Errors: every call returns a qp_status; qp_last_error() returns a thread-local
 *     message with a one-line remedy. No call aborts the process.
 *   - There is no CPU fallback: device entry points fail with QP_ERR_CUDA when no
 *     sm_100 device is present.
 *   - Widths (bits_x4 = 4 * bits per weight; Table 1, plus uniform SQ):
 *       QP_TCQ       1.5 .. 5.0  step 0.5   (bits_x4 6,8,..,20; shift s = 2b)
 *       QP_HALF_TCQ  1.75 .. 4.75 step 0.5  (bits_x4 7,9,..,19; d_in halves at b, b+0.5)
 *       QP_VQ        1.5 .. 6.0  step 0.5   (bits_x4 6,8,..,24; 2b-bit index per pair)
 *       QP_NUQ       2 .. 8                 (bits_x4 8,12,..,32)
 *       QP_UNIF      2 .. 8                 (bits_x4 8,12,..,32)
 *     others -> QP_ERR_UNSUPPORTED_WIDTH.
 *   - Partition (else QP_ERR_PARTITION_MISMATCH): d_out % 32 == 0, d_in % 256 == 0,
 *     half-TCQ also (d_in / 2) % 256 == 0; batch in 1..8 ("batch sizes up to 8").
 */
#ifndef QPALETTE_H
#define QPALETTE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  QP_OK = 0,
  QP_ERR_INVALID_ARG = 1,        /* null pointer, negative size, bad enum            */
  QP_ERR_UNSUPPORTED_WIDTH = 2,  /* scheme/bits_x4 not in Table 1             */
  QP_ERR_PARTITION_MISMATCH = 3, /* shapes not multiples of the tile         */
  QP_ERR_DIM = 4,                /* incompatible dimensions                   */
  QP_ERR_CONFIG_MISMATCH = 5,    /* codebook / rotation do not match the layer*/
  QP_ERR_LENGTH = 6,             /* byte count does not match the layout     */
  QP_ERR_ALLOC = 7,              /* device allocation failed                         */
  QP_ERR_CUDA = 8,               /* CUDA runtime error (incl. no sm_100 device)      */
  QP_ERR_NCCL = 9,               /* NCCL error                                       */
  QP_ERR_UNSUPPORTED = 10        /* valid request this build does not implement      */
} qp_status;

typedef enum { QP_NUQ = 0, QP_UNIF = 1, QP_VQ = 2, QP_TCQ = 3, QP_HALF_TCQ = 4 } qp_scheme;
typedef enum { QP_F16 = 0, QP_BF16 = 1, QP_F32 = 2 } qp_dtype;

/* flags of the forward calls */
#define QP_X_PREROTATED 1u   /* x is already R x in fp16 (skip the rotation kernel) */
#define QP_NO_PDL 2u         /* launch without programmatic dependent launch        */
#define QP_DETERMINISTIC 4u  /* fp32 y: in-order cross-CTA reduction (bitwise reproducible) instead of
                                zero-then-atomic-add (fp16 y is always in-order)        */
#define QP_FUSE_RHT 16u    /* compute R x inside the GEMV kernel (every CTA, in shared memory; fp32 y
                                zeroed in-kernel) instead of launching the rotation kernel, when x'
                                fits the kernel's plan. Opt-in: on B200 at the C2 shapes the
                                PDL-overlapped rotation kernel is faster (profiles/r1/ab_xs_r1.md) */
#define QP_INDEPENDENT 32u  /* qp_multi_fwd only: no work still running on the stream reads or writes this
                                call's x or y (e.g. independent requests, or steps whose inputs are already
                                resident): the engine launch then does not wait for the preceding kernel
                                (griddepcontrol.wait), only for the previous launch of the same qp_multi,
                                so consecutive calls overlap. Ignored by the per-layer fallback.        */
#define QP_Y_ACCUMULATE 8u  /* fp32 y only: y += diag(s) W_hat R x (y is not zeroed first; e.g. a residual
                                add). Not with QP_DETERMINISTIC.                                        */

typedef struct qp_codebook qp_codebook;
typedef struct qp_rht qp_rht;
typedef struct qp_layer qp_layer;
typedef struct qp_group qp_group;
typedef struct qp_multi qp_multi;

/* Route the library's device allocations (e.g. to PyTorch's caching allocator).
 * alloc(size, ctx) returns a device pointer or NULL; free_(ptr, ctx). Pass NULLs to
 * restore cudaMalloc/cudaFree. Must be called before objects are created. */
qp_status qp_set_allocator(void* (*alloc)(size_t, void*), void (*free_)(void*, void*), void* ctx);

/* Load a frozen fp16 codebook (host memory, little-endian IEEE half, row-major).
 *   QP_TCQ / QP_HALF_TCQ: tlut [2^tb][2] of TCQ at the (upper) width, tb = 9 for b <= 4,
 *        10 for 4.5, 11 for 5.0; the hybrid LUT is quantlut_sym(tlut, L, tb)
 *        (P:1025-1033), L in {12, 16} (L = 16 is the paper's; 12 is config C1).
 *   QP_VQ: LUT [2^(2b)][2].   QP_NUQ / QP_UNIF: LUT [2^b].
 * n_bytes must equal the table size (else QP_ERR_LENGTH). L is ignored for non-TCQ. */
qp_status qp_codebook_load(qp_scheme scheme, int bits_x4, int L, const void* host_fp16, size_t n_bytes,
                           qp_codebook** out);
void qp_codebook_free(qp_codebook* cb);

/* Reconstruction scale alpha of a TCQ codebook at its width (reading R22: "appropriate
 * scaling", made rate-dependent so that TCQ stays close to the distortion bound at
 * every width). The frozen tlut keeps unit second moment; the offline quantizers divide
 * the standardized weights by alpha and store the scales s * alpha, so decode is unchanged.
 * Values: codebooks/tcq_alpha.json (written by scripts/calibrate_tcq_alpha.py from oracle/).
 * Default 1. Set it before quantizing. Errors: QP_ERR_INVALID_ARG (NULL, alpha <= 0 / not finite). */
qp_status qp_codebook_set_scale(qp_codebook* cb, double alpha);

/* Rotation R for inputs of width d_in. block = 0 selects the largest
 * power-of-two divisor of d_in; otherwise block must be a power of two dividing d_in. */
qp_status qp_rht_create(uint64_t seed, int d_in, int block, qp_rht** out);
void qp_rht_free(qp_rht* r);

/* x_rot[batch][d_in] (fp16, device) = R x (x device, [batch][d_in] of dtype xt).
 * Arithmetic in fp32, one rounding to fp16 at the end. */
qp_status qp_rht_apply(const qp_rht* r, const void* x, qp_dtype xt, int batch, void* x_rot, void* stream);

/* Layer from packed codes (host, LAYOUT.md order, exactly d_out*d_in*bits/8 bytes) and
 * fp32 per-output-channel scales (host, d_out). Copies both to the device. */
qp_status qp_layer_from_codes(const void* codes_host, size_t n_bytes, const float* scales_host, int d_out, int d_in,
                              qp_scheme scheme, int bits_x4, const qp_codebook* cb, const qp_rht* r, qp_layer** out);

/* Data-free quantization of an nn.Linear weight W[d_out][d_in] (host fp32, row-major)
 * (P:348): W' = W R^T, s_j = RMS(W'_j), W~ = W'/s, then RTN (NUQ, UNIF, VQ) or the
 * rotate-half tail-biting Viterbi (TCQ, half-TCQ; reading R4), on n_threads
 * host threads (0 = all). Host-side and slow at L = 16 (~0.1 s per 256-weight trellis per
 * thread): use qp_quantize_offline_gpu for TCQ layers of real size. */
qp_status qp_quantize_offline(const float* W_host, int d_out, int d_in, qp_scheme scheme, int bits_x4,
                              const qp_codebook* cb, const qp_rht* r, int n_threads, qp_layer** out);

/* qp_quantize_offline with the TCQ / half-TCQ trellis search on the current GPU:
 * every (tile, lane) trellis is one CTA's rotate-half Viterbi in float64 with the host
 * encoder's operation order, so the codes are bitwise those of qp_quantize_offline (rotation,
 * scales, RTN schemes and bit packing stay on the host). Synchronous; allocates device scratch
 * (~0.5 MB per SM at L = 16). Errors as qp_quantize_offline, plus QP_ERR_CUDA. */
qp_status qp_quantize_offline_gpu(const float* W_host, int d_out, int d_in, qp_scheme scheme, int bits_x4,
                                  const qp_codebook* cb, const qp_rht* r, int n_threads, qp_layer** out);

/* Copy a layer's codes / scales back to the host (n_bytes must equal the stored size). */
qp_status qp_layer_get_codes(const qp_layer* l, void* codes_host, size_t n_bytes);
qp_status qp_layer_get_scales(const qp_layer* l, float* scales_host);

/* y[batch][d_out] (device, dtype yt in {F16, F32}) = diag(s) W_hat R x (the fused
 * dequantize-and-multiply). x: device [batch][d_in] of dtype xt, or R x in
 * fp16 with QP_X_PREROTATED. Two kernels: rotation (+ zeroing of fp32 y) and the fused GEMV,
 * PDL-chained; with QP_FUSE_RHT one kernel when x' fits its shared-memory plan (every CTA computes
 * R x itself -- bitwise the rotation kernel's x' -- and zeroes fp32 y in-kernel). */
qp_status qp_linear_fwd(const qp_layer* l, const void* x, qp_dtype xt, int batch, void* y, qp_dtype yt,
                        unsigned flags, void* stream);

/* Fused group: members share d_in, rotation, scheme, width and codebook
 * (e.g. q/k/v or up/gate). One GEMV launch over the concatenated rows; ys[i] receives
 * member i's rows ([batch][d_out_i]). Members are copied; they may be freed afterwards. */
qp_status qp_fuse(const qp_layer* const* members, int n, qp_group** out);
void qp_group_free(qp_group* g);
qp_status qp_fused_linear(const qp_group* g, const void* x, qp_dtype xt, int batch, void* const* ys, qp_dtype yt,
                          unsigned flags, void* stream);

/* W_hat[d_out][d_in] (device fp16) without scales: the dequantization-only kernel
 * (P:1154-1163). Bit-exact against the oracle's decode (frozen fp16 codebooks). */
qp_status qp_dequantize(const qp_layer* l, void* W_hat_fp16, void* stream);

/* Persistent multi-layer engine: y_i = diag(s_i) W_hat_i R_i x_i for a list of n independent
 * layers (P:345-362 per layer), run as ONE persistent launch per run of consecutive layers that
 * share a decode table (e.g. TCQ widths 2.5-4.0 on the tb = 9 tlut, or one VQ / NUQ width): the
 * activation rotations run inside the launch (device-side ready flags instead of a kernel
 * boundary), the replicated table is built once, every layer's tiles form one stream-K range over
 * all SMs, and split row tiles reduce through a self-cleaning fp32 workspace (no zeroing kernel).
 * Layers without an engine variant run through qp_linear_fwd inside qp_multi_fwd.
 * qp_multi_create references (does not own) the layers: free the qp_multi first. It allocates the
 * per-layer scratch (x' 16*d_in B, workspace 32*d_out B, counters) once, so qp_multi_fwd never
 * allocates and is graph-capturable. A qp_multi may be used by one stream at a time.
 * qp_multi_fwd: xs[i] device [batch][d_in_i] of dtype xt (16-byte aligned; with QP_X_PREROTATED fp16
 * R x, 32-byte aligned), ys[i] device [batch][d_out_i] of dtype yt in {F16, F32}; outputs must not
 * alias inputs. Flags: QP_X_PREROTATED, QP_NO_PDL, QP_Y_ACCUMULATE (fp32 y += ...), QP_INDEPENDENT. QP_DETERMINISTIC
 * and QP_FUSE_RHT are rejected (QP_ERR_INVALID_ARG). Other errors as qp_linear_fwd. */
qp_status qp_multi_create(const qp_layer* const* layers, int n, qp_multi** out);
qp_status qp_multi_fwd(qp_multi* m, const void* const* xs, qp_dtype xt, int batch, void* const* ys, qp_dtype yt,
                       unsigned flags, void* stream);
/* Row-sharded qp_multi_fwd (north star: large layers row-sharded over the node, all-gather of y):
 * the qp_multi's layers are this rank's shards (qp_layer_shard with the communicator's world size);
 * the engine computes every shard's rows, then ONE grouped ncclAllGather (ncclGroupStart / End)
 * assembles ys_full[i] [batch][d_out_i * world] (dtype yt) on every rank, ranks' rows in rank order.
 * Errors: as qp_multi_fwd, QP_ERR_CONFIG_MISMATCH (a layer is not a shard of this world size),
 * QP_ERR_NCCL (incl. an asynchronous NCCL fault of an earlier call); QP_Y_ACCUMULATE is rejected. */
qp_status qp_multi_fwd_sharded(qp_multi* m, const void* const* xs, qp_dtype xt, int batch, void* const* ys_full,
                               qp_dtype yt, void* comm, unsigned flags, void* stream);
/* Row-sharded multi-layer forward with the all-gather FUSED into the engine epilogue (north star's
 * all-gather step): every layer of m is this rank's row shard (qp_layer_shard; m_i =
 * d_out_i rows); each final y value of this rank's rows is stored by the engine directly into every
 * rank's y_full of that layer over peer-mapped memory (NVLink), at [b][rank * m_i + row] of the
 * [batch][world * m_i] layout, so no collective kernel, gather scratch or permutation follows.
 * ys_peers[i * world + k]: rank k's y_full of layer i (dtype yt, mapped with qp_ipc_open; this rank's
 * own at k = rank), laid out identically on every rank: layer i's buffer at the same byte offset from
 * layer 0's on every rank (QP_ERR_INVALID_ARG otherwise); flag_peers[k]: rank k's flag array (unsigned[2 * world + 1], zeroed once), as in
 * qp_linear_fwd_sharded_p2p, whose y_full reuse rule applies (a rank stores round n into a peer's
 * y_full only after that peer entered round n). Each engine launch of the call is one round, with the
 * entry announcement, the entry gate, the delivery and the wait for every rank's delivery inside the
 * kernel: the launch completes once every rank's rows of its layers have arrived. Every layer
 * must have an engine variant (QP_ERR_UNSUPPORTED otherwise); QP_Y_ACCUMULATE / QP_INDEPENDENT are
 * rejected (QP_ERR_INVALID_ARG). A peer that never arrives traps the wait kernel after 20 s. */
qp_status qp_multi_fwd_sharded_p2p(qp_multi* m, const void* const* xs, qp_dtype xt, int batch,
                                   void* const* ys_peers, unsigned* const* flag_peers, int rank, int world,
                                   qp_dtype yt, unsigned flags, void* stream);
/* n_layers; launch groups per qp_multi_fwd (n_launches: one engine launch each, or the per-layer
 * qp_linear_fwd path for a layer without an engine variant); how many are engine launches. */
qp_status qp_multi_info(const qp_multi* m, int* n_layers, int* n_launches, int* n_engine_launches);
void qp_multi_free(qp_multi* m);

/* Contiguous row block [rank*d_out/world, (rank+1)*d_out/world) of a layer as a new
 * layer (device copy). (d_out/world) % 32 must be 0. */
qp_status qp_layer_shard(const qp_layer* l, int rank, int world, qp_layer** out);

/* Column (k) shard for row-parallel layers (the down projection after a column-parallel
 * up / gate): rank r owns input columns [r*d_in/world, (r+1)*d_in/world) of every row (a new layer of
 * shape d_out x d_in/world holding those k tiles, all scales, and its own rotation = the blocks of R
 * over its columns, which is exact because R is block-diagonal, P:345-349 / reading R9). Needs
 * (d_in/world) % 256 == 0 and % rotation block == 0 (QP_ERR_PARTITION_MISMATCH otherwise: quantize
 * with a smaller block via qp_rht_create(seed, d_in, block)); half-TCQ -> QP_ERR_UNSUPPORTED. */
qp_status qp_layer_shard_k(const qp_layer* l, int rank, int world, qp_layer** out);

/* K-sharded forward: y[batch][d_out] (device fp32) = sum over ranks of diag(s) W_r R_r x_r, where
 * x_local = this rank's columns x[:, r*d_in/world : ...] ([batch][d_in/world], dtype xt): the shard's
 * partial GEMV, then ncclAllReduce(sum) over `comm`. QP_Y_ACCUMULATE is rejected; asynchronous NCCL
 * faults surface as QP_ERR_NCCL. */
qp_status qp_linear_fwd_ksharded(const qp_layer* shard, const void* x_local, qp_dtype xt, int batch, void* y,
                                 qp_dtype yt, void* comm, unsigned flags, void* stream);

/* Host-only (no device work, usable without a GPU): where rank `rank` of `world` finds its row
 * shard of a (d_out x d_in, scheme, bits_x4) layer: rows [*row0, *row0 + *rows) and code bytes
 * [*byte0, *byte0 + *nbytes) of the LAYOUT.md stream (row-tile-major, so a row block is one
 * contiguous byte range). The all-gather of qp_linear_fwd_sharded concatenates the ranks' rows in
 * rank order. Errors: QP_ERR_INVALID_ARG (NULL / rank outside [0, world)),
 * QP_ERR_UNSUPPORTED_WIDTH, QP_ERR_PARTITION_MISMATCH (d_out % world, (d_out/world) % 32, or the
 * layer's own partition rules). */
qp_status qp_shard_range(int d_out, int d_in, qp_scheme scheme, int bits_x4, int rank, int world, int* row0,
                         int* rows, size_t* byte0, size_t* nbytes);

/* Host-only (no device work): Theorem 1 of the paper, the optimal fractional bit
 * allocation with ideal Gaussian quantizers for L layers with sensitivities a[l] > 0 and sizes
 * n[l] = d_in * d_out > 0 (weights) under a total budget of M bits and a floor eta:
 *     b_out[l] = max{eta, ln(a[l] / n[l]) / (2 ln 2) + C},  C such that sum_l b_out[l] n[l] = M.
 * Exact (sorted breakpoints, no iteration). The caller owns all arrays (length L).
 * Errors: QP_ERR_INVALID_ARG (NULL, L <= 0, non-positive a / n, eta < 0),
 * QP_ERR_CONFIG_MISMATCH (infeasible: M < eta * sum n). */
qp_status qp_optimal_bits(const double* a, const double* n, int L, double M, double eta, double* b_out);

/* Host-only: fusion-aware mixed-scheme quantization, solved exactly. For n_blocks
 * Transformer blocks with layers (q, k, v, o, u, g, d), sensitivities a[b*7 + l], quantizer
 * distortions err[q] (data-free loss a_l * err_q) and profiled latencies cost[t*n_quant
 * + q] of group type t in (q, k, v, qk, qv, kv, qkv, o, u, g, ug, d) quantized by q, choose the
 * fusible groups and one quantizer per group minimising the total loss with total cost <= budget
 * (fusion = 0: singleton groups only, the plain MSQ of P:436-440). Outputs per layer b*7 + l: the
 * group type it belongs to (group_out) and its quantizer (quant_out); optional totals. Exact
 * multiple-choice-knapsack solution by Pareto frontiers. Errors: QP_ERR_INVALID_ARG,
 * QP_ERR_CONFIG_MISMATCH (budget below the cheapest assignment), QP_ERR_ALLOC (frontier > 4 M). */
qp_status qp_plan_msq(int n_blocks, const double* a, int n_quant, const double* err, const double* cost,
                      double budget, int fusion, int* group_out, int* quant_out, double* loss_out, double* cost_out);

/* NCCL plumbing for the row-sharded path (NCCL over NVLink / NVSwitch).
 * qp_nccl_unique_id writes 128 bytes; broadcast them (e.g. with torch.distributed)
 * and call qp_nccl_comm_create on every rank. comm is an ncclComm_t. */
qp_status qp_nccl_unique_id(void* id128);
qp_status qp_nccl_comm_create(const void* id128, int world, int rank, void** comm);
qp_status qp_nccl_comm_destroy(void* comm);

/* Row-sharded forward: this rank computes its shard's rows, then an all-gather over
 * `comm` assembles y_full[batch][d_out_full] (device, dtype yt) on every rank. */
qp_status qp_linear_fwd_sharded(const qp_layer* shard, const void* x, qp_dtype xt, int batch, void* y_full,
                                qp_dtype yt, void* comm, unsigned flags, void* stream);

/* Row-sharded forward with the all-gather fused into the GEMV epilogue (peer
 * memory over NVLink / NVSwitch instead of ncclAllGather): every final y value of this rank's rows
 * is stored directly into all `world` ranks' y_full ([batch][world * shard_d_out], dtype yt in
 * {F16, F32}, rank r's rows at columns [r*m, (r+1)*m)); then the grid's last CTA increments this
 * rank's counter in every rank's flag array, and a one-thread wait kernel on `stream` returns once
 * every rank has delivered into this rank's y_full, so later work on `stream` sees the whole
 * vector. y_peers[k] / flag_peers[k]: rank k's y_full and flag array (unsigned[2 * world + 1], zeroed
 * once at setup, mapped into this process with qp_ipc_open; this rank's own pointers at k = rank).
 * Buffer reuse: each call first runs a round-entry barrier (every rank announces the round in all
 * flag arrays and waits for the others), so a rank stores round n into a peer's y_full only after
 * that peer has *entered* round n -- i.e. its work on y_full enqueued on `stream` before this call is
 * done. Readers of y_full must therefore be ordered before the next call on the same stream.
 * Uses the in-order (QP_DETERMINISTIC) epilogue; QP_Y_ACCUMULATE / QP_FUSE_RHT are rejected.
 * Errors: QP_ERR_INVALID_ARG, plus qp_linear_fwd's. Graph-capturable (no host-side epoch). */
qp_status qp_linear_fwd_sharded_p2p(const qp_layer* shard, const void* x, qp_dtype xt, int batch,
                                    void* const* y_peers, unsigned* const* flag_peers, int rank, int world,
                                    qp_dtype yt, unsigned flags, void* stream);

/* The permutation qp_linear_fwd_sharded applies after ncclAllGather for batch > 1: src [world][batch][m]
 * (rank-major, as the all-gather delivers it) -> dst [batch][world * m] (device buffers, elem_bytes 2 or
 * 4, no aliasing). Exposed for callers that run their own all-gather, and for tests. */
qp_status qp_gather_permute(const void* src, void* dst, int world, int batch, int m, int elem_bytes, void* stream);

/* CUDA IPC plumbing for qp_linear_fwd_sharded_p2p. qp_ipc_handle writes 72 bytes: the 64-byte CUDA
 * IPC handle of the allocation that contains dev_ptr (found with cuMemGetAddressRange: dev_ptr may
 * lie inside a caching-allocator segment) + the 8-byte offset of dev_ptr in it. qp_ipc_open maps a
 * peer's handle into this process (peer access enabled lazily) and returns the peer's dev_ptr;
 * qp_ipc_close unmaps it. Errors: QP_ERR_INVALID_ARG (NULL), QP_ERR_CUDA. */
qp_status qp_ipc_handle(const void* dev_ptr, void* handle72);
qp_status qp_ipc_open(const void* handle72, void** dev_ptr);
qp_status qp_ipc_close(void* dev_ptr);

/* Introspection. bits_per_weight counts code bits only (reading R19). */
qp_status qp_layer_info(const qp_layer* l, size_t* code_bytes, double* bits_per_weight, int* d_out, int* d_in);

/* Number of kernels the library has enqueued since load (for launch accounting). */
uint64_t qp_launch_count(void);

void qp_layer_free(qp_layer* l);
const char* qp_last_error(void);
const char* qp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QPALETTE_H */
