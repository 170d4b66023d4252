/*
 * decdec.h -- C ABI of the B200-native DecDEC decode hot path.
 *
 * DecDEC (arXiv 2412.20185) augments every decode-step linear layer (a GEMV) with
 * dynamic error compensation:
 *
 *     o = W_hat x + sum_{i in S(x)} x_i * R_hat[i, :]
 *
 *   (1) S(x) = indices of the k largest |x_i|                     (P:207 step 1, "Exact")
 *   (2) fetch R_hat[S, :] (4-bit residual codes + per-column scales) from pinned host
 *       memory with GPU zero-copy loads over PCIe                  (P:207 step 2)
 *   (3) o_dec = x[S]^T R_hat[S, :]                                 (P:207 step 3)
 *   (4) o = o_b + o_dec, o_b = W_hat x the base GEMV               (P:207 step 4)
 *
 * Conventions (all entry points):
 *   - Pointers are plain device / host pointers; no framework types.  "device" means
 *     CUDA global memory of the current device; "host mapped" means memory returned by
 *     decdec_host_alloc (or cudaHostAlloc(..., cudaHostAllocMapped)).
 *   - Ownership: the caller owns every buffer.  The library never allocates on the hot
 *     path.  The workspace is caller-provided, reusable across layers, one per
 *     concurrently used stream, and must be zeroed once (decdec_workspace_init) before
 *     its first use; every successful call leaves it ready for the next call.
 *   - Errors: arguments are validated synchronously; on error nothing is enqueued and a
 *     negative decdec_status is returned.  Launch failures return DECDEC_ECUDA.
 *     Asynchronous device faults surface at the next stream synchronisation.
 *   - fp16 values are passed as uint16_t bit patterns (IEEE binary16).
 *   - Shapes: d_in % 128 == 0 (group size 128), 128 <= d_in <= 32768,
 *     d_out % 32 == 0 (16-byte residual rows), d_out >= 32.
 *   - Determinism: results are bit-identical run to run (no value atomics; fixed
 *     accumulation orders).
 */
#ifndef DECDEC_H_
#define DECDEC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* decdec_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  DECDEC_OK = 0,
  DECDEC_EINVAL = -1,       /* bad shape / k / chunk / null pointer                        */
  DECDEC_EALIGN = -2,       /* pointer not 16-byte aligned                                */
  DECDEC_ENOTMAPPED = -3,   /* residual pointer is not host-mapped (zero-copy) memory      */
  DECDEC_EUNSUPPORTED = -4, /* bits / r_bits / d_in outside the supported set              */
  DECDEC_ECUDA = -5,        /* CUDA runtime error (allocation, launch, attribute)          */
  DECDEC_ENCCL = -6,        /* reserved for the library-owned communicator path            */
  DECDEC_ESPACE = -7        /* workspace or output buffer too small                        */
} decdec_status;

#define DECDEC_GROUP 128

/*
 * One quantized linear layer (or this rank's output-column shard of one).
 *
 * Base weights W_hat = s * (q - z), RTN asymmetric, groups of 128 input channels per
 * output column (DESIGN.md ledger L5; stands in for AWQ).  Packed K-major:
 * output column j is a contiguous row of its d_in codes (ledger L6):
 *   w_bits = 4 (layout W4K): uint32 [d_out][d_in/8]; channel c of an 8-channel word at
 *            bit 4*(c>>1) + 16*(c&1).
 *   w_bits = 3 (layout W3K): uint32 [d_out][3*d_in/32]; per 32-channel slice 3 words:
 *            channel c < 30 -> word c/10, bits 16*h + 3*p .. +2 with r = c%10, p = r/2,
 *            h = r%2; channels 30/31 -> code bit b at word b, bit 15 (+16 for c = 31).
 *            3.0 bits per weight.
 * w_format = DECDEC_WFMT_LUT (the paper's non-uniform base, SqueezeLLM served by a LUT kernel,
 * P:397): W_hat[i][j] = w_lut[j][q_ij], codes q < 2^w_bits
 * (w_bits = 3 | 4) packed as W4K nibbles (4 bits per weight for both widths), no s / z
 * (w_scales / w_zeros unused).  Tables: fp16 [d_out][2^w_bits].  Compensation (k > 0) runs
 * in the same fused kernel (rows' tables staged in place of the scales) with r_bits = 4 only;
 * r_bits = 16 on a LUT layer: DECDEC_EUNSUPPORTED.
 * Residual R_hat = S_j * c_ij, c in [-7, 7]: rows = input channels,
 * contiguous, in HOST MAPPED memory (zero-copy):
 *   r_bits = 4  (layout Rq):  uint32 [d_in][d_out/8], nibble = c + 8, column c of an
 *            8-column word at bit 4*(c>>1) + 16*(c&1); r_scales fp16 [d_out] (host mapped,
 *            fetched on every call).
 *   r_bits = 16 (layout R16): fp16 [d_in][d_out] (Table 3 "FP16"); r_scales NULL.
 */
#define DECDEC_WFMT_UNIFORM 0 /* W3K / W4K codes + fp16 s + u8 z per 128-group (AWQ-style RTN)   */
#define DECDEC_WFMT_LUT 1     /* non-uniform: W4K nibble codes < 2^w_bits + per-column fp16 table */

typedef struct decdec_layer {
  int32_t d_in, d_out;       /* d_out = this rank's shard width when sharded             */
  int32_t w_bits;            /* 3 | 4                                                    */
  int32_t group_size;        /* must be 128                                              */
  const void* w_packed;      /* device, 16-B aligned, W3K | W4K                           */
  const uint16_t* w_scales;  /* device fp16 [d_out][d_in/128], 16-B aligned               */
  const uint8_t* w_zeros;    /* device u8   [d_out][d_in/128], 16-B aligned               */
  int32_t r_bits;            /* 4 (paper default) | 16                                   */
  const void* r_rows;        /* HOST mapped, 16-B aligned, Rq | R16                       */
  const uint16_t* r_scales;  /* HOST mapped fp16 [d_out] (r_bits = 4) | NULL (r_bits = 16) */
  int32_t w_format;          /* DECDEC_WFMT_UNIFORM (0, default) | DECDEC_WFMT_LUT (1)       */
  const uint16_t* w_lut;     /* LUT: device fp16 [d_out][2^w_bits], 16-B aligned; else unused */
} decdec_layer;

/* Bytes of workspace for layers with k <= max_k and d_out <= max_d_out: a reserved 16 KB
 * head, then the fp32 base output o_b (d_out) handed from the GEMV CTAs to the
 * deterministic combine.  Every o_b entry is self-validating: it holds the pattern
 * 0xFFFFFFFF (a NaN no arithmetic produces) until the GEMV stores it, and the combine
 * restores the pattern after reading it, so no fence or arrival counter is needed.
 * (The paper's k x (4+2) B sc_indices / x[sc_indices] buffer lives in the shared
 * memory of each DEC CTA; max_k does not change the size, it is kept for ABI stability.)
 * A workspace serves one stream at a time; layers on that stream may share it. */
size_t decdec_workspace_bytes(int32_t max_k, int32_t max_d_out);

/* Initialise a workspace (stream-ordered): head zeroed, o_b set to the empty pattern.
 * Required once before first use. */
decdec_status decdec_workspace_init(void* ws, size_t ws_bytes, decdec_stream_t stream);

/*
 * decdec_linear: y = fp16_rn( W_hat x + sum_{i in S} x_i R_hat[i,:] ), one decode step
 * of one layer.  x, y: device fp16 [d_in] / [d_out], 16-B aligned.
 *   chunk = 0    : S = exact global Top-k of |x| ("Exact"); 0 <= k <= d_in.
 *   chunk = 1024 : the paper's chunk partition made exact and deterministic:
 *                  in every contiguous 1024-channel chunk the top min(k, len) channels,
 *                  here k = k_chunk <= 1024 (total = sum over chunks).
 *   Magnitude = 15-bit key bits(x) & 0x7FFF; ties -> lower index (ledger L2).  x must be
 *   finite (NaN/Inf: undefined).
 *   k = 0 runs the plain quantized GEMV, bit-identical to decdec_gemv.
 *   sel: optional device int32 output receiving the selected indices ascending
 *        (S:119); capacity >= total selected.  May be NULL.
 * Enqueues on `stream`; asynchronous.
 */
decdec_status decdec_linear(const decdec_layer* L, const uint16_t* x, int32_t k, int32_t chunk,
                            uint16_t* y, int32_t* sel, void* ws, size_t ws_bytes,
                            decdec_stream_t stream);

/* Plain quantized GEMV y = fp16_rn(W_hat x) (the uncompensated baseline, k = 0). */
decdec_status decdec_gemv(const decdec_layer* L, const uint16_t* x, uint16_t* y, void* ws,
                          size_t ws_bytes, decdec_stream_t stream);

/* Step (1) alone: exact Top-k (S:117-131 exact_topk).  idx: device int32 [n_sel],
 * xs: device fp16 [n_sel]; n_sel = k (chunk = 0) or sum_c min(k, len_c) (chunk > 0).
 * x: device fp16 [d_in], 16-B aligned, d_in % 8 == 0, d_in <= 32768 (else DECDEC_EINVAL /
 * DECDEC_EALIGN; idx 4-B and xs 2-B aligned). */
decdec_status decdec_select(const uint16_t* x, int32_t d_in, int32_t k, int32_t chunk,
                            int32_t* idx, uint16_t* xs, decdec_stream_t stream);

/* Number of channels selected for (d_in, k, chunk); -1 on invalid arguments. */
int32_t decdec_num_selected(int32_t d_in, int32_t k, int32_t chunk);

/* ------------------------------------------------------------------ native step executor */
/* A decode step's sequence of layer calls captured once into a CUDA graph (one stream,
 * layer i+1 after layer i; inside a layer the selector and the fused kernel overlap via
 * programmatic dependent launch).  Buffers x[i], y[i] and the shared workspace are
 * bound at creation; replays read whatever those buffers hold.  All layers are validated
 * before capture; on error nothing is created.  chunk applies to every layer; k[i] is the
 * per-layer k (or k_chunk when chunk > 0). */
typedef struct decdec_stack decdec_stack;
decdec_status decdec_stack_create(const decdec_layer* layers, int32_t n_layers, const int32_t* k, int32_t chunk,
                                  const uint16_t* const* x, uint16_t* const* y, void* ws, size_t ws_bytes,
                                  decdec_stream_t stream, decdec_stack** out);
decdec_status decdec_stack_launch(decdec_stack* s, decdec_stream_t stream);
int32_t decdec_stack_kernels(const decdec_stack* s); /* kernels per launch, -1 if NULL */
void decdec_stack_destroy(decdec_stack* s);

/* ------------------------------------------------------------------ tensor parallelism */
/* Output-feature sharding (BASELINE.json north_star "the layer shards by
 * output features ... output assembled with an NCCL all-gather over NVLink").  Rank r holds
 * columns [r*d_out_r, (r+1)*d_out_r) of W_hat (its device memory) and of R_hat + scales (its
 * own pinned host slice behind its own PCIe link); x is replicated, so every rank selects the
 * identical S (exact, deterministic selector; ledger L11) and no index exchange is needed.
 * The communicator is library-owned; NCCL is loaded at run time (dlopen of libnccl.so.2,
 * reusing one already loaded in the process).  Errors: DECDEC_ENCCL if NCCL cannot be loaded
 * or a NCCL call fails. */
typedef struct decdec_comm decdec_comm;

/* NCCL version code of the loaded library (e.g. 22809), -1 if NCCL cannot be loaded. */
int32_t decdec_nccl_version(void);

/* Fill id_out (128 bytes, host) with a new NCCL unique id.  Call on one rank and broadcast
 * the bytes to the others out of band (e.g. the torch.distributed process group). */
decdec_status decdec_nccl_unique_id(void* id_out);

/* Collective over all nranks: create this rank's communicator on the current device. */
decdec_status decdec_comm_init(const void* id, int32_t rank, int32_t nranks, decdec_comm** out);
void decdec_comm_destroy(decdec_comm* c);
int32_t decdec_comm_rank(const decdec_comm* c);   /* -1 if NULL */
int32_t decdec_comm_nranks(const decdec_comm* c); /* -1 if NULL */

/* decdec_linear on this rank's shard L (L->d_out = d_out_r), writing its outputs straight
 * into y_full + rank*d_out_r, followed on the same stream by an in-place all-gather that
 * leaves the full y (device fp16 [nranks*d_out_r], 16-B aligned) on every rank.  Every rank
 * must call it with the same x, k, chunk and d_out_r.  sel/ws as decdec_linear. */
decdec_status decdec_linear_tp(const decdec_layer* L, const uint16_t* x, int32_t k, int32_t chunk,
                               uint16_t* y_full, int32_t* sel, void* ws, size_t ws_bytes, decdec_comm* comm,
                               decdec_stream_t stream);

/* A TP decode step captured as one CUDA graph: for each layer i, decdec_linear on the shard
 * into y_full[i] + rank*d_out_r(i), then the in-place all-gather of y_full[i]
 * ([nranks*layers[i].d_out]).  Launch/destroy with decdec_stack_launch/_destroy. */
decdec_status decdec_stack_create_tp(const decdec_layer* layers, int32_t n_layers, const int32_t* k, int32_t chunk,
                                     const uint16_t* const* x, uint16_t* const* y_full, void* ws, size_t ws_bytes,
                                     decdec_comm* comm, decdec_stream_t stream, decdec_stack** out);

/* ---- fused P2P-store all-gather (the exchange inside the layer
 * kernel's epilogue instead of a separate collective).  Each rank owns a symmetric device
 * region: a flag area (1024 per-layer completion counters) and a user area of user_bytes
 * holding the y_full buffers, at the same offsets on every rank.  The layer kernel stores its
 * shard's fp16 outputs into EVERY rank's y_full through CUDA-IPC peer mappings (NVLink stores
 * on a multi-GPU node), releases one count per writing CTA to every rank's flag of the layer's
 * slot, and completes only after this rank's flag shows all nranks' shards (acquire, system
 * scope).  The launch is cooperative (every CTA co-resident), so the wait cannot starve the
 * writers.  Ranks may share one GPU (separate processes; the driver time-slices them). */
typedef struct decdec_peers decdec_peers;
#define DECDEC_IPC_HANDLE_BYTES 64

/* This rank's region on the current device (zeroed); handle_out (64 bytes, host) receives its
 * IPC handle, to be exchanged with the other ranks out of band (e.g. the torch process group).
 * Errors: DECDEC_EINVAL (NULL args), DECDEC_ECUDA (allocation / IPC export failed). */
decdec_status decdec_peers_create(size_t user_bytes, void* handle_out, decdec_peers** out);
/* Open every other rank's region; handles = nranks x 64 bytes in rank order (this rank's own
 * entry is ignored).  1 <= nranks <= 8, once per group.  DECDEC_ECUDA if a handle cannot be
 * opened (no peer access between the devices). */
decdec_status decdec_peers_connect(decdec_peers* p, int32_t rank, int32_t nranks, const void* handles);
/* Device address / size of this rank's user area (NULL / 0 if p is NULL). */
void* decdec_peers_buffer(const decdec_peers* p);
size_t decdec_peers_buffer_bytes(const decdec_peers* p);
void decdec_peers_destroy(decdec_peers* p);

/* decdec_linear on this rank's shard L (d_out_r = L->d_out) whose outputs land at byte offset
 * y_off of EVERY rank's user area: y_full = buffer + y_off, fp16 [nranks*d_out_r], this rank's
 * shard at y_full + rank*d_out_r.  On return (stream order) y_full is complete on this rank.
 * slot (0..1023) names the completion counter; calls that may overlap in time across ranks
 * (consecutive layers) need distinct slots, and every rank must issue the same sequence of
 * (slot, shape, k, chunk).  y_off must be 16-B aligned and y_off + nranks*d_out_r*2 <= user
 * bytes.  sel/ws as decdec_linear.  Errors as decdec_linear; DECDEC_EINVAL if the peer group is
 * not connected or slot/y_off are out of range; DECDEC_EUNSUPPORTED for LUT-base layers. */
decdec_status decdec_linear_p2p(const decdec_layer* L, const uint16_t* x, int32_t k, int32_t chunk, size_t y_off,
                                int32_t slot, int32_t* sel, void* ws, size_t ws_bytes, decdec_peers* peers,
                                decdec_stream_t stream);

/* A TP decode step with the fused all-gather, captured as one CUDA graph: layer i as
 * decdec_linear_p2p(layers[i], x[i], k[i], chunk, y_off[i], slot = i) (n_layers <= 1024). */
decdec_status decdec_stack_create_p2p(const decdec_layer* layers, int32_t n_layers, const int32_t* k, int32_t chunk,
                                      const uint16_t* const* x, const size_t* y_off, void* ws, size_t ws_bytes,
                                      decdec_peers* peers, decdec_stream_t stream, decdec_stack** out);

/* ---- multi-link residual fetch (the analogue of the paper's GH200
 * C2C observation): when peer GPUs are idle (no tensor parallelism), a layer's
 * residual gather is split across their PCIe links.  Every rank of a decdec_peers group calls
 * decdec_linear_ml with the same layer (same packed residual contents in its own host-mapped
 * memory; the base weights are read on rank 0 only), x, k and chunk.  Every rank computes the
 * identical selection S; rank r fetches the positions p of S with p % nranks == r, and the helper
 * ranks (r > 0) store their o_dec parts (fp32, times S_j) into rank 0's user area over NVLink;
 * rank 0 runs the base GEMV, its own share, and adds the helpers' parts in rank order before
 * writing y.  Handshake per DEC CTA (flag + ack words in the user area at ml_off, the same
 * offset on every rank, decdec_ml_bytes(d_out, nranks) bytes): a helper writes only after rank 0
 * consumed its previous part, so consecutive calls need no other synchronisation.  y / sel are
 * rank 0's (helpers: ignored, may be NULL).  k = 0 or a single rank: rank 0 runs decdec_linear
 * alone and helpers return at once.  Errors as decdec_linear; DECDEC_EINVAL (group not
 * connected, ml_off not 16-B aligned), DECDEC_ESPACE (ml area outside the user area),
 * DECDEC_EUNSUPPORTED (more than 64 DEC CTAs).  A peer that never arrives traps after ~20 s. */
size_t decdec_ml_bytes(int32_t d_out, int32_t nranks);
decdec_status decdec_linear_ml(const decdec_layer* L, const uint16_t* x, int32_t k, int32_t chunk, uint16_t* y,
                               int32_t* sel, void* ws, size_t ws_bytes, decdec_peers* peers, size_t ml_off,
                               decdec_stream_t stream);

/* ------------------------------------------------------------------ offline, host-only */
/* Pack base codes q (u8 [d_in][d_out], logical W layout, values < 2^bits) into W3K/W4K
 * (uint32 [d_out][d_in*bits/32]).  out_bytes must be >= d_out*d_in*bits/8. */
decdec_status decdec_pack_weights(const uint8_t* q, int32_t d_in, int32_t d_out, int32_t bits,
                                  void* out, size_t out_bytes);

/* Pack residual codes c (int8 [d_in][d_out], values in [-7, 7]) into Rq
 * (uint32 [d_in][d_out/8]).  out_bytes >= d_in*d_out/2. */
decdec_status decdec_pack_residual(const int8_t* c, int32_t d_in, int32_t d_out, void* out,
                                   size_t out_bytes);

/* Pinned, device-mapped host memory for the residual store (zero-copy source).
 * numa_node >= 0 binds the pages to that node before pinning; -1 = no binding.
 * write_combined != 0 requests write-combined pages (GPU reads only). */
decdec_status decdec_host_alloc(size_t bytes, int32_t numa_node, int32_t write_combined, void** p);
void decdec_host_free(void* p);

/* NUMA node of a CUDA device's PCIe attachment (/sys/bus/pci/devices/<bdf>/numa_node), for
 * binding each rank's residual slice to the socket in front of its own PCIe link (SURVEY.md
 * §8(e)); -1 when unknown (no NUMA, bad device).  Host-only, no GPU work. */
int32_t decdec_device_numa_node(int32_t device);

/* ------------------------------------------------------------------ debug / introspection */
/* Decode the packed weights with the GEMV kernel's own in-register decode path and write
 * the integer codes to q_out (device u8 [d_out][d_in]).  For bit-exact layout tests. */
decdec_status decdec_debug_unpack_weights(const decdec_layer* L, uint8_t* q_out,
                                          decdec_stream_t stream);

/* Debug timelines: while buf != NULL every launch records %globaltimer (ns) / SM-cycle events
 * into buf (u64: [0..1] unused, then per CTA 20 events, see csrc/linear.cuh kTraceEvents:
 * 0 start, 2 x loaded, 3 first stage landed, 4 GEMV done, 5 selector start, 6 selection
 * published, 7 gather done, 9 combine done, 10 last warp exits, 12 partials published, 14-19
 * selector phases in SM cycles; DEC CTAs come first).  Single calls: bytes >= (2 + 1024*20)*8.
 * Stacks created while tracing give layer i the region starting at u64 2 + i*160*20; their
 * creation fails with DECDEC_ESPACE unless bytes >= (2 + n_layers*3200)*8.  Not thread-safe;
 * NULL disables. */
decdec_status decdec_debug_trace(void* buf, size_t bytes);

/* Debug (tests): while idx != NULL, every DEC CTA c < max_ctas of each compensated launch
 * (the CTAs that select, gather and combine; each computes the selection itself)
 * writes its own selected indices / x[S] in its placement order (a permutation of the
 * ascending selection) to idx[c*cap ...] / xs[c*cap ...] (device int32 / fp16, at most cap
 * entries each).  Lets tests check EVERY DEC CTA's selection bit-exact, not only the `sel`
 * output of CTA 0.  idx = NULL disables.  DECDEC_EINVAL if cap or max_ctas <= 0.  Not
 * thread-safe; process-wide. */
decdec_status decdec_debug_selections(int32_t* idx, uint16_t* xs, int32_t cap, int32_t max_ctas);

/* Launch plan chosen for a layer (tile rows, consumer warps, stages, grid) as text. */
decdec_status decdec_plan_string(const decdec_layer* L, int32_t k, char* buf, size_t buf_bytes);

/* Tuning knob (the paper's n_tb; §4.4 tuner): number of DEC CTAs -- CTAs of
 * the fused layer kernel that select, gather and combine -- used by layer calls planned after
 * this call (decdec_linear, decdec_stack_create*).  0 (default) = automatic; the plan may
 * double it when shared memory requires.  1 <= n <= 64.  Process-wide, not thread-safe. */
decdec_status decdec_set_dec_ctas(int32_t n);

/* Number of kernels decdec_linear enqueues for (k): always 1 (the selector runs on the fused
 * kernel's first CTA(s)). */
int32_t decdec_launches_per_call(int32_t k);

const char* decdec_status_string(decdec_status s);
const char* decdec_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DECDEC_H_ */
