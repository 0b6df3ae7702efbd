/*
 * sagips.h -- C ABI of libsagips.so, the B200 (sm_100a) implementation of the
 * data-parallel hot path of SAGIPS (arXiv 2407.00051): the per-rank GAN
 * training step of the proxy inverse problem and the asynchronous ring
 * exchange of generator weight gradients with grouping.
 *
 * Citations: P:<n> = line n of the paper's LaTeX source;
 * R<n> = a reading recorded in DESIGN.md where the paper is silent.
 *
 * Conventions (apply to every call below)
 *  - One context per rank, one rank per GPU.  The caller selects the device
 *    (cudaSetDevice) before sagips_create and before every call.
 *  - "dev" pointers are CUDA device pointers, "host" pointers are host
 *    memory.  The caller owns every pointer it passes; the library keeps
 *    device pointers into the workspace the caller gave to sagips_create,
 *    which must outlive the context.  The library itself owns only the host
 *    context, its CUDA events/graphs/NCCL communicator, and (multi-rank
 *    only) one cudaMalloc'ed exchange window that it exports by IPC handle.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Calls marked [async] only enqueue work on that stream;
 *    calls marked [sync] return after their work is complete.
 *  - Every call returns a sagips_status and never aborts or exits.  On
 *    failure sagips_last_error(ctx) returns a message.  An asynchronous
 *    device-side failure (a non-finite loss, an exchange timeout) is
 *    reported by the next [sync] call.
 *  - Every floating-point buffer is IEEE fp32, row-major.
 */
#ifndef SAGIPS_H
#define SAGIPS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SAGIPS_ABI_VERSION 1

#if defined(__GNUC__)
#define SAGIPS_API __attribute__((visibility("default")))
#else
#define SAGIPS_API
#endif

typedef enum {
  SAGIPS_OK = 0,
  SAGIPS_ERR_INVALID_ARG = 1,  /* NULL pointer, size mismatch, bad `which` */
  SAGIPS_ERR_CONFIG = 2,       /* inconsistent sagips_config (see sagips_create) */
  SAGIPS_ERR_CUDA = 3,         /* a CUDA runtime / driver error */
  SAGIPS_ERR_NONFINITE = 4,    /* a loss became NaN/Inf (the SPEC's NaN guard) */
  SAGIPS_ERR_PROTOCOL = 5,     /* exchange packet tag mismatch */
  SAGIPS_ERR_STATE = 6,        /* call out of order (e.g. pull before push) */
  SAGIPS_ERR_TIMEOUT = 7,      /* an exchange wait exceeded its bound */
  SAGIPS_ERR_UNSUPPORTED = 8   /* feature not built / not available */
} sagips_status;

/* Gradient-exchange modes, Tab. III plus the two reference
 * points of the paper's study. */
typedef enum {
  SAGIPS_MODE_NONE = 0,           /* ensemble: no exchange */
  SAGIPS_MODE_ARAR = 1,           /* ungrouped ring over all ranks */
  SAGIPS_MODE_ARAR_ARAR = 2,      /* inner ring (two-sided) + outer ring every h */
  SAGIPS_MODE_RMA_ARAR_ARAR = 3,  /* inner ring one-sided (RMA) + outer ring */
  SAGIPS_MODE_SYNC_ALLREDUCE = 4, /* synchronous all-reduce sum (the Horovod role) */
  SAGIPS_MODE_RMA_ALLGATHER = 5,  /* as RMA_ARAR_ARAR, but the inner group exchanges by a one-hop
                                     all-gather over NVSwitch: every member stores its packet into
                                     every other member's window (no pass-along); same sums (§8(f) row 3) */
  SAGIPS_MODE_RMA_CHUNKED = 6     /* as RMA_ARAR_ARAR with staleness 0 only: the inner group's sum as a
                                     one-sided chunked reduce-scatter + all-gather (member q folds chunk
                                     q of every packet in ascending origin order and stores the result
                                     into every member's window): 2 (g-1)/g packets per rank instead
                                     of g - 1, the same sums (the paper's future work) */
} sagips_mode;

typedef enum {
  SAGIPS_PREC_FP32 = 0,  /* fp32-class (R20, R28): CUDA-core layers in fp32; the 128 -> 128
                            discriminator GEMMs on tcgen05 with bf16-split operands x = hi + lo,
                            fp32 accumulation -- forward/dgrad hi*hi + hi*lo + lo*hi (bf16x3),
                            wgrad G_hi*H_hi + G_lo*H_hi (bf16x2); everything else fp32 */
  SAGIPS_PREC_BF16 = 1   /* discriminator GEMMs bf16 x bf16 -> fp32 on tcgen05, fp32 master weights */
} sagips_precision;

typedef enum {
  SAGIPS_DISC_AUTO = 0,     /* tcgen05 for 128-wide hidden layers, else CUDA-core fp32 */
  SAGIPS_DISC_SIMT = 1,     /* CUDA-core FFMA everywhere (fp32 only) */
  SAGIPS_DISC_TCGEN05 = 2   /* tcgen05 (requires disc_hidden == 128); FP32 precision runs bf16x3 */
} sagips_disc_impl;

typedef enum {
  SAGIPS_PRESET_DESK = 0,  /* C1: G [8,64,64,6], D [2,64,64,1], k=64, m=16 */
  SAGIPS_PRESET_PAPER = 1  /* C2: G [6,128x4,6], D [2,128x4,1] (51,206 / 50,049 params), k=1024, m=1024 */
} sagips_preset;

typedef enum {
  SAGIPS_SAMPLER_QUADRATIC = 0,  /* Q(u; c) = c0 + c1 u + c2 u^2 (R1) */
  SAGIPS_SAMPLER_TABULATED = 1   /* density on a grid, tabulated CDF, binary-search inversion (R32) */
} sagips_sampler;

typedef struct {
  /* ranks and exchange */
  int32_t world;          /* number of ranks (GPUs) */
  int32_t rank;           /* this rank, 0..world-1 */
  int32_t group_size;     /* inner group size g: contiguous groups of g ranks, the last one may be
                             smaller; leaders = first rank of each group;
                             g == world: ungrouped */
  int32_t outer_every;    /* h: leaders' ring fires when (step+1) % h == 0; 0 = never (R13) */
  int32_t mode;           /* sagips_mode */
  int32_t staleness;      /* s in {0,1}: other members' packets from step t-s (R12); 0 for RMA_CHUNKED */
  int32_t reduce_mean;    /* 1: divide the reduced packet by the number of contributors (R11) */
  int32_t precision;      /* sagips_precision for the discriminator GEMMs */
  /* model dimensions (R4, R5) */
  int32_t noise_dim;      /* d */
  int32_t gen_hidden;     /* generator hidden width */
  int32_t gen_depth;      /* number of generator hidden layers */
  int32_t disc_hidden;    /* discriminator hidden width */
  int32_t disc_depth;     /* number of discriminator hidden layers */
  /* batch (Tab. IV) */
  int32_t param_samples;      /* k: generator rows per step */
  int32_t events_per_sample;  /* m: events drawn per parameter sample; N = k*m */
  int64_t reference_rows;     /* N_ref: loop-closure reference events */
  int64_t shard_rows;         /* n_s: this rank's bootstrap shard (50%) */
  /* optimisation (R7) */
  float gen_lr, disc_lr, leaky_slope, adam_beta1, adam_beta2, adam_eps;
  /* loop closure: true parameters in constrained space (R3) */
  float true_params[6];
  /* diagnostic histograms (R22) */
  int32_t hist_bins;
  float hist_lo[2], hist_hi[2];
  uint64_t seed;              /* Philox key (R-RNG) */
  int32_t exchange_timeout_ms;/* bound on every exchange wait (0 = 10000) */
  int32_t phase_timing;       /* 1: record CUDA events at the phase boundaries of every step */
  int32_t disc_impl;          /* sagips_disc_impl: kernels of the discriminator hidden layers */
  int32_t sampler;            /* sagips_sampler of a3-a9: the closed-form quadratic quantile (R1,
                                 default) or the tabulated CDF (R32); with the
                                 latter, true_params holds (w, b, c) per observable, w in (0,1),
                                 b, c > 0, and the reference data are drawn with it */
  int32_t sampler_grid;       /* G of the tabulated sampler, 3..2048 (0 = 1024) */
  int32_t packet_biases;      /* 1: tensor fusion: the exchanged packet
                                 is [weights | biases] and Adam(G) applies the reduced bias
                                 gradients; 0 (default): weights only, biases local */
  int32_t outer_rma;          /* one-sided modes only: 1 = the leaders' outer ring (R13) also runs
                                 through the exchange windows (one-hop all-gather of the leaders'
                                 inner sums over NVLink, no NCCL); 0 (default) = NCCL send/recv,
                                 the paper's two-sided ARAR outer group (Tab. III) */
  int32_t reserved[1];
} sagips_config;

typedef struct sagips_ctx sagips_ctx;

/* What sagips_get / sagips_set / sagips_tensor_bytes address.  Shapes use
 * k = param_samples, N = k*m, Pw = generator weights-only count (packet),
 * Pb = generator bias count, Qw/Qb = discriminator weights/biases. */
typedef enum {
  SAGIPS_T_GEN_W = 0,        /* [Pw]  generator weights, layer order, each W_l[out][in] row-major */
  SAGIPS_T_GEN_B = 1,        /* [Pb]  generator biases, layer order */
  SAGIPS_T_DISC_W = 2,       /* [Qw]  discriminator weights */
  SAGIPS_T_DISC_B = 3,       /* [Qb]  discriminator biases */
  SAGIPS_T_GEN_ADAM = 4,     /* [2(Pw+Pb)] Adam state m_W[Pw], v_W[Pw], m_b[Pb], v_b[Pb] */
  SAGIPS_T_DISC_ADAM = 5,    /* [2(Qw+Qb)] m_W[Qw], v_W[Qw], m_b[Qb], v_b[Qb] */
  SAGIPS_T_NOISE = 6,        /* [k][d]  generator input of the last step */
  SAGIPS_T_RAW = 7,          /* [k][6]  generator output */
  SAGIPS_T_C = 8,            /* [k][6]  constrained coefficients (c0,c1,c2) per observable */
  SAGIPS_T_EVENTS = 9,       /* [2N][2] discriminator input: rows 0..N-1 real, N..2N-1 fake */
  SAGIPS_T_REAL_IDX = 10,    /* [N] uint32 bootstrap indices into the shard */
  SAGIPS_T_HIST = 11,        /* [2 real/fake][2 obs][bins+2] uint32 */
  SAGIPS_T_LOGITS_D = 12,    /* [2N] discriminator logits of the D step */
  SAGIPS_T_LOGITS_G = 13,    /* [N]  logits of the G step (updated D) */
  SAGIPS_T_DY = 14,          /* [N][2] dL_G / d events */
  SAGIPS_T_DRAW = 15,        /* [k][6] dL_G / d raw */
  SAGIPS_T_GEN_DW = 16,      /* [Pw] local generator weight gradient = the packet */
  SAGIPS_T_GEN_DB = 17,      /* [Pb] local generator bias gradient */
  SAGIPS_T_DISC_DW = 18,     /* [Qw] discriminator weight gradient of the D step */
  SAGIPS_T_DISC_DB = 19,     /* [Qb] */
  SAGIPS_T_REDUCED = 20,     /* [Pw] reduced packet applied to the generator ([Pw + Pb] with packet_biases) */
  SAGIPS_T_STATS = 21,       /* sagips_step_stats of the last step */
  SAGIPS_T_REFERENCE = 22,   /* [N_ref][2] reference events */
  SAGIPS_T_SHARD = 23,       /* [n_s][2] this rank's shard */
  SAGIPS_T_COUNT = 24
} sagips_tensor;

typedef struct {
  float loss_d;          /* L_D of the step (mean over 2N rows, R9) */
  float loss_g;          /* L_G (mean over N rows) */
  uint64_t step;         /* step index of the last completed train_step */
  uint32_t outer_fired;  /* 1 if the leaders' ring ran this step */
  uint32_t nonfinite;    /* 1 if a loss was NaN/Inf */
  uint64_t wait_ns;      /* time spent waiting for peer packets (exchange) */
  uint64_t reserved[4];
} sagips_step_stats;

/* train_step flags */
#define SAGIPS_STEP_LOCAL_ONLY  1u  /* run steps a1-a11 (through the packet) only; no exchange, no Adam(G) */
#define SAGIPS_STEP_NO_ADAM_G   2u  /* exchange but do not apply the generator update */
#define SAGIPS_STEP_GRAPH       4u  /* capture the step's launches into a CUDA graph and replay it as one
                                       graph launch (the executable graph is updated in place from step
                                       to step; host-input steps, sagips_train_step_host, included);
                                       ignored on the first step, on steps whose outer ring fires on this
                                       rank (they run eagerly) and for the two-sided ring modes (ARAR,
                                       ARAR_ARAR), whose pull waits on an earlier step's side-stream
                                       ring.  Phase / kernel timing is not recorded for graph steps.
                                       The one-sided pass-along ring joins its forwarding agent into
                                       the step at the end of a graph step. */

/* Fill *cfg with a preset (sagips_preset) on world=1, rank=0, mode NONE,
 * seed 1, lr 1e-5/1e-4, Adam (0.9, 0.999, 1e-8), slope 0.01, the
 * true parameters (1, 1, 0.5, 2, 0.5, 1) (R3), 64 bins over [0,4). [sync]
 * Errors: INVALID_ARG for a NULL cfg or an unknown preset. */
SAGIPS_API sagips_status sagips_config_init(sagips_config* cfg, int32_t preset);

/* Device bytes the caller must provide to sagips_create for cfg. [sync]
 * Errors: INVALID_ARG (NULL), CONFIG (as sagips_create). */
SAGIPS_API sagips_status sagips_workspace_size(const sagips_config* cfg, size_t* bytes);

/* Create the rank context on the current device.  `workspace` is a device
 * buffer of >= sagips_workspace_size bytes (256-byte aligned), owned by the
 * caller.  Initialises, on `stream`: the generator with Kaiming-normal
 * weights identical on every rank, this rank's discriminator,
 * the reference data from the true parameters (identical on every
 * rank = rank 0's data distribution, R19) and this rank's 50%
 * bootstrap shard. [sync]
 * Errors: CONFIG if the generator output is not 6 (Eq. 4) or D is not 2->1,
 * group_size < 1, staleness not in {0,1}, mode unknown, outer_rma not in
 * {0,1}, or a constrained true parameter c1/c2 <= 0; CUDA on device errors. */
SAGIPS_API sagips_status sagips_create(const sagips_config* cfg, void* workspace, size_t workspace_bytes,
                            void* stream, sagips_ctx** out);

/* Frees the context and, for world > 1, the exchange window that peers map.
 * The caller must quiesce the ranks first: every rank synchronises its
 * streams and passes a barrier (e.g. torch.distributed.barrier) before any
 * rank calls destroy, so no peer store into this window is in flight
 * (runtime.close does this). [sync] */
SAGIPS_API sagips_status sagips_destroy(sagips_ctx* ctx);
SAGIPS_API const char* sagips_last_error(const sagips_ctx* ctx);
SAGIPS_API int32_t sagips_abi_version(void);

/* Standalone inverse-CDF sampler (R1): for e in [0, k*m), s = e/m,
 * o in {0,1}: u = uniform(word 2e+o of Philox stream (step, rank, stream_id))
 * (R-RNG, R-UNIF) and events[e][o] = c0 + u*(c1 + u*c2) in fp32, each
 * operation rounded separately, with (c0,c1,c2) = c[s][3o..3o+2].
 * c: dev [k][6] constrained coefficients.  events: dev [k*m][2].
 * hist: dev [2][bins+2] uint32 (zeroed here) or NULL: index 0 underflow
 * (and NaN), 1..bins the bins of [lo[o], hi[o]), bins+1 overflow (R22).
 * lo, hi: host float[2].  [async]
 * Errors: INVALID_ARG for NULL c/events, k<1, m<1, bins<1 with hist. */
SAGIPS_API sagips_status sagips_sample_events(const float* c, int32_t k, int32_t m, uint64_t seed,
                                   uint64_t step, uint32_t rank, uint32_t stream_id,
                                   float* events, uint32_t* hist, int32_t bins,
                                   const float* lo, const float* hi, void* stream);

/* Tabulated-CDF sampler variant (reading R32;
 * the inverse-CDF method of P:295 on a tabulated density): for parameter
 * sample s and observable o, (w, b, c) = (sigmoid(r0), softplus(r1),
 * softplus(r2)) of (r0, r1, r2) = raw[s][3o..3o+2] and the density
 * f(x) = w x^b (1-x)^c + (1-w) x^c (1-x)^b on [0, 1], tabulated on G nodes
 * t_i = i/(G-1) with a trapezoid CDF F_i = S_i / S_{G-1} (fp64); event e of
 * sample s = e / m: events[e][o] = t_i + (u - F_i) / (F_{i+1} - F_i) / (G-1)
 * for the cell i with F_i <= u < F_{i+1}, u = uniform(word 2e+o of Philox
 * stream (step, rank, stream_id)) as in sagips_sample_events.  raw: dev
 * [k][6] fp32; events: dev [k*m][2] fp32; 3 <= G <= 2048.  [async]
 * Errors: INVALID_ARG (NULL, k < 1, m < 1, G out of range, k*m >= 2^31). */
SAGIPS_API sagips_status sagips_sample_tabulated(const float* raw, int32_t k, int32_t m, int32_t G, uint64_t seed,
                                                 uint64_t step, uint32_t rank, uint32_t stream_id, float* events,
                                                 void* stream);
/* Its backward (R32): draw[s][3o+j] = dtheta_j/dr_j * sum over the sample's
 * events of dy[e][o] dx_e/dtheta_j, the exact derivative of the tabulated
 * inverse (theta = (w, b, c)); the same u as the forward; fixed-order fp64
 * sums.  dy: dev [k*m][2] fp32; draw: dev [k][6] fp32.  [async]
 * Errors: as sagips_sample_tabulated, and NULL dy / draw. */
SAGIPS_API sagips_status sagips_sample_tabulated_bwd(const float* raw, int32_t k, int32_t m, int32_t G, uint64_t seed,
                                                     uint64_t step, uint32_t rank, uint32_t stream_id,
                                                     const float* dy, float* draw, void* stream);

/* Generator prediction G(n) (the G_i(n) of Eq. 7): the constrained
 * parameters c = constrain(G(noise)) (R1) of this rank's current generator
 * for a caller-given noise batch, for the ensemble analysis.
 * noise: dev [k][noise_dim] fp32; c_out: dev [k][6] fp32, row s = c of noise
 * vector s; 1 <= k <= cfg.param_samples.  Call between training steps: it
 * reuses the step's generator activation buffers (the next step recomputes
 * them).  [async]  Errors: INVALID_ARG (NULL, k out of range), UNSUPPORTED
 * (a generator layer wider than 128). */
SAGIPS_API sagips_status sagips_predict_params(sagips_ctx* ctx, const float* noise, int32_t k, float* c_out,
                                               void* stream);

/* Ensemble response and normalised residuals (§8(f) rows 2 and 4): preds is
 * dev [M][k][P] fp32, preds[i][s][j] = parameter j predicted by ensemble
 * member i for noise vector s.  out (host, 3P doubles):
 *   out[j]        p_hat_j = (1/k) sum_s (1/M) sum_i preds[i][s][j]   (Eq. 7)
 *   out[P + j]    sigma_j = (1/k) sum_s sqrt((1/M) sum_i (preds[i][s][j] - mean_s)^2)  (Eq. 8)
 *   out[2P + j]   r_hat_j = (p_true[j] - p_hat_j) / p_true[j]   (Eq. 6; NaN if p_true is NULL)
 * p_true: host [P] doubles or NULL.  Sums in fp64 in a fixed order
 * (deterministic).  M, k >= 1, 1 <= P <= 16.  [sync]  Errors: INVALID_ARG;
 * CUDA. */
SAGIPS_API sagips_status sagips_ensemble_stats(const float* preds, int32_t M, int32_t k, int32_t P,
                                               const double* p_true, double* out, void* stream);

/* One training step t of this rank: noise -> G -> constrain ->
 * sampler -> bootstrap real batch -> D step + Adam(D) -> G loss through the
 * updated D -> backprop through the sampler and G -> weights-only packet
 * and then, unless SAGIPS_STEP_LOCAL_ONLY, push + pull (exchange per
 * cfg.mode) + Adam(G).  Steps are consecutive: t = previous t + 1 (the first
 * call may use any t, except 0 in exchanging modes with staleness 1, whose
 * pull(t) needs the peers' packets of t - 1). [async]
 * Errors: STATE if t is not the next step; TIMEOUT / PROTOCOL if an earlier
 * exchange wait of this rank failed (reported by the next call without a
 * sync; that step's fold and Adam(G) were skipped, so the generator keeps
 * its weights); CUDA. */
SAGIPS_API sagips_status sagips_train_step(sagips_ctx* ctx, uint64_t step, uint32_t flags, void* stream);

/* sagips_train_step with the step's inputs supplied by the caller (host
 * memory, pinned for asynchronous copies), for a data-loading pipeline: the
 * generator noise of a1 (host_noise: [k][noise_dim] fp32, else drawn by
 * Philox) and the real batch of a5 (host_real: [N][2] fp32 real rows,
 * replacing the bootstrap from the resident shard; the real half of the
 * histogram is then zero and SAGIPS_T_REAL_IDX is not written).  They are
 * copied on a library-owned stream into one of two device staging buffers
 * of the workspace (slot step & 1), which `stream` waits for, so a caller
 * that issues step t+1 before waiting for step t overlaps t+1's host-to-
 * device copy with t's compute; the host buffers must stay unchanged until
 * the step's stats are valid.  host_stats (or NULL) receives the step's
 * stats record by an asynchronous copy at its end (valid once `stream` has
 * completed).  [async]  Errors: as sagips_train_step. */
SAGIPS_API sagips_status sagips_train_step_host(sagips_ctx* ctx, uint64_t step, uint32_t flags,
                                                const float* host_noise, const float* host_real,
                                                sagips_step_stats* host_stats, void* stream);

/* Exchange halves, for callers that overlap them with other work.  push
 * publishes the step-t packet to the ring (one-sided: a store into the
 * successor's window + release flag; two-sided: NCCL send/recv).
 * pull waits (bounded by exchange_timeout_ms) for the packets it needs,
 * forwards the ring, folds in ascending origin order (R10), applies the
 * outer ring when it fires (R13) and runs Adam(G). [async]
 * One-sided modes: pull is a one-warp wait kernel (only one thread spins)
 * followed by the fold + Adam(G) kernel (programmatic dependent launch); if
 * the wait times out or finds an overrun slot, the fold and Adam(G) are
 * skipped on the device and the error is returned by the next call.
 * Errors: STATE if pull(t) precedes push(t) or train_step(t, LOCAL_ONLY);
 * TIMEOUT / PROTOCOL as sagips_train_step. */
SAGIPS_API sagips_status sagips_push_generator_grad(sagips_ctx* ctx, uint64_t step, void* stream);
SAGIPS_API sagips_status sagips_pull_generator_grad(sagips_ctx* ctx, uint64_t step, void* stream);

/* Copy a tensor to / from host memory.  `bytes` must equal
 * sagips_tensor_bytes(which).  [sync]  Errors: INVALID_ARG; SAGIPS_T_STATS
 * with a non-finite flag returns NONFINITE after copying. */
SAGIPS_API sagips_status sagips_tensor_bytes(const sagips_ctx* ctx, int32_t which, size_t* bytes);
SAGIPS_API sagips_status sagips_get(sagips_ctx* ctx, int32_t which, void* host, size_t bytes);
SAGIPS_API sagips_status sagips_set(sagips_ctx* ctx, int32_t which, const void* host, size_t bytes);

/* Multi-rank plumbing (world > 1).  The exchange window is cudaMalloc'ed by
 * the library.  Every rank exports its handle (64 bytes, cudaIpcMemHandle_t)
 * and then connects to all ranks' handles gathered by the caller (e.g.
 * torch.distributed.all_gather_object) in rank order. [sync] */
#define SAGIPS_IPC_HANDLE_BYTES 64
SAGIPS_API sagips_status sagips_ipc_handle(sagips_ctx* ctx, void* host_handle, size_t bytes);
SAGIPS_API sagips_status sagips_connect_peers(sagips_ctx* ctx, const void* host_handles, size_t bytes);

/* Single-process wiring (several contexts of one process on one device, e.g.
 * W emulated ranks in a test; CUDA IPC cannot open a handle in the process
 * that exported it): sagips_window_ptr returns the device address of this
 * context's exchange window (0 if the mode has none); after every context
 * has one, sagips_connect_peers_local takes the world's window addresses in
 * rank order (n == world) instead of IPC handles.  The one-sided modes then
 * behave exactly as across processes (same kernels, same release/acquire
 * tags).  The caller orders the launches so that no kernel waits on work
 * queued behind it on the same stream (e.g. all LOCAL_ONLY steps, then all
 * pushes, then all pulls). [sync]  Errors: INVALID_ARG (NULL, n != world,
 * own address mismatch), STATE (already connected). */
SAGIPS_API sagips_status sagips_window_ptr(sagips_ctx* ctx, uint64_t* dev_ptr);
SAGIPS_API sagips_status sagips_connect_peers_local(sagips_ctx* ctx, const uint64_t* dev_ptrs, size_t n);

/* NCCL (two-sided ring and the synchronous all-reduce).  Rank 0 creates the
 * id (128 bytes, ncclUniqueId), the caller broadcasts it, every rank
 * connects. [sync]  Errors: UNSUPPORTED if built without NCCL. */
#define SAGIPS_NCCL_ID_BYTES 128
SAGIPS_API sagips_status sagips_nccl_unique_id(void* host_id, size_t bytes);
SAGIPS_API sagips_status sagips_connect_nccl(sagips_ctx* ctx, const void* host_id, size_t bytes);

/* Phases of a step, in order: 0 noise + generator forward + constrain
 * (a1-a3), 1 sampler + bootstrap + histograms (a4-a6), 2 discriminator step
 * incl. Adam(D) (a7), 3 generator loss through the updated D back to dy
 * (a8), 4 sampler backward (a9), 5 generator backward -> packet (a10-a11),
 * 6 exchange + Adam(G) (a12-a13). */
#define SAGIPS_NUM_PHASES 7
/* Mean device time (ms, CUDA events on the step stream) of each phase over
 * the last min(steps, 64) steps run with cfg.phase_timing = 1.  host_ms has
 * n >= SAGIPS_NUM_PHASES floats. [sync]  Errors: STATE if timing is off. */
SAGIPS_API sagips_status sagips_phase_times(sagips_ctx* ctx, float* host_ms, int32_t n, int32_t* steps_averaged);

/* Tensor-core discriminator kernels of a step (paper widths, depth >= 3),
 * in launch order: 0 D forward first layer, 1 D forward middle layer(s), 2 D
 * forward last hidden layer + head + BCE, 3 D backward layer L-2 (wgrad +
 * dgrad), 4 D backward middle layer(s), 5 D backward first layer (+ layer-0
 * gradients); 6-11 the same for the G step (no wgrad; 11 yields dy); 12 the
 * fused G step (k_gstep: all layers of the G step in one kernel, activations
 * in tensor memory -- it replaces 6-11, depth 4); 13 the fused D forward
 * (k_dfwd: layers 0-3 + head, replaces 0-2).  Mean device ms per step (CUDA
 * events on the step stream around each launch; a class with several
 * launches, e.g. middle layers, sums them) over the last min(steps, 64) steps
 * run with cfg.phase_timing = 1; host_ms has n >= SAGIPS_NUM_KERNELS floats;
 * unused classes are 0. [sync]  Errors: STATE if timing is off or no step
 * ran. */
#define SAGIPS_NUM_KERNELS 14
SAGIPS_API sagips_status sagips_kernel_times(sagips_ctx* ctx, float* host_ms, int32_t n, int32_t* steps_averaged);
/* Forget the recorded phase / kernel times (e.g. after warm-up steps, whose
 * first launches include lazy module loading). [sync] */
SAGIPS_API sagips_status sagips_timing_reset(sagips_ctx* ctx);

/* Debugging aid: with the environment variable SAGIPS_TRACE=1 set before the
 * first step, the tensor-core layer kernels record globaltimer stamps per
 * tile (CTAs 0-3, first 32 launches): [launch][cta][tile][4] uint64 =
 * producer done, MMA start, epilogue start, epilogue done, followed by
 * [launch][256 CTAs][12] uint64 per-CTA records: start and end stamps (0, 1)
 * and, for the per-layer kernels, summed wait times in ns (4 + k: k = 1
 * loader slot, 2 MMA operands, 3 MMA accumulator, 4 producers' slot, 5
 * epilogue accumulator, 6 mask flag, 7 epilogue X rows).  Copies and rearms
 * the buffer; `bytes` must equal the size returned for host == NULL.
 * [sync] */
SAGIPS_API sagips_status sagips_debug_trace(void* host, size_t* bytes);

/* CUDA-graph steps (SAGIPS_STEP_GRAPH): graph launches and graph
 * instantiations (an instantiation happens when the step's topology changes,
 * e.g. the first steps of staleness 1) since create. [sync] */
SAGIPS_API sagips_status sagips_graph_stats(const sagips_ctx* ctx, uint64_t* graph_launches, uint64_t* instantiations);

/* Number of this library's kernels launched since create (all streams;
 * kernels inside a captured graph step count once, at capture). */
SAGIPS_API sagips_status sagips_launch_count(const sagips_ctx* ctx, uint64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* SAGIPS_H */
