// sagips.cu -- the C ABI of libsagips.so (include/sagips.h): rank context,
// workspace layout in HBM, and the stream-ordered orchestration of one
// SAGIPS training step (order R8).
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sagips.h"
#include "ctx.h"
#include "internal.h"

namespace sagips {

static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
uint64_t launches_total() { return g_launches.load(std::memory_order_relaxed); }

void MlpLayout::build(int in, int hidden, int depth, int out) {
  L = depth + 1;
  sizes[0] = in;
  for (int i = 1; i <= depth; ++i) sizes[i] = hidden;
  sizes[L] = out;
  nw = nb = 0;
  maxw = 0;
  for (int l = 0; l < L; ++l) {
    w_off[l] = nw;
    b_off[l] = nb;
    nw += (int64_t)sizes[l + 1] * sizes[l];
    nb += sizes[l + 1];
    maxw = std::max(maxw, std::max(sizes[l], sizes[l + 1]));
  }
}

// ---------------------------------------------------------------- layout
// All device buffers are carved out of the caller's workspace (256-B
// aligned).  The same function sizes (base == nullptr) and carves.
struct Carver {
  char* base;
  size_t off = 0;
  template <typename T>
  T* take(int64_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += sizeof(T) * (size_t)std::max<int64_t>(count, 1);
    return p;
  }
};

static int wgrad_splits(int M, int N, int64_t K) {
  const int tiles = ((M + 127) / 128) * ((N + 127) / 128);
  int s = std::max(1, 296 / tiles);
  const int64_t kmax = std::max<int64_t>(1, K / 256);
  return (int)std::min<int64_t>(s, kmax);
}

static void carve(sagips_ctx* c, char* base) {
  Carver cv{base};
  const sagips_config& g = c->cfg;
  const int64_t k = g.param_samples, N = c->N;
  auto& G = c->G;
  auto& D = c->D;
  c->gW = cv.take<float>(G.nw);  c->gB = cv.take<float>(G.nb);
  c->gmW = cv.take<float>(G.nw); c->gvW = cv.take<float>(G.nw);
  c->gmB = cv.take<float>(G.nb); c->gvB = cv.take<float>(G.nb);
  c->dW = cv.take<float>(D.nw);  c->dB = cv.take<float>(D.nb);
  c->dmW = cv.take<float>(D.nw); c->dvW = cv.take<float>(D.nw);
  c->dmB = cv.take<float>(D.nb); c->dvB = cv.take<float>(D.nb);
  c->g_dW = cv.take<float>(G.nw + G.nb); c->g_dB = c->g_dW + G.nw;  // contiguous: the fused packet
  c->d_dW = cv.take<float>(D.nw); c->d_dB = cv.take<float>(D.nb);
  c->reduced = cv.take<float>(G.nw + G.nb);
  c->ref = cv.take<float>(2 * g.reference_rows);
  c->shard = cv.take<float>(2 * g.shard_rows);
  c->noise = cv.take<float>(k * g.noise_dim);
  for (int l = 0; l < G.L; ++l) c->gAct[l] = cv.take<float>(k * G.sizes[l + 1]);
  c->gdZ[0] = cv.take<float>(k * G.maxw);
  c->gdZ[1] = cv.take<float>(k * G.maxw);
  for (int l = 0; l + 1 < G.L; ++l) c->gdz_all[l] = cv.take<float>(k * G.sizes[l + 1]);
  c->cbuf = cv.take<float>(6 * k);
  c->draw = cv.take<float>(6 * k);
  c->X = cv.take<float>(4 * N);
  c->real_idx = cv.take<uint32_t>(N);
  // rows rounded up to whole 128-row tiles (plane-tile format, k_tc_layers.cu)
  const int64_t rows_t = (2 * N + 127) / 128 * 128;
  for (int l = 0; l < D.L - 1; ++l) c->dAct[l] = cv.take<float>(rows_t * D.sizes[l + 1]);
  for (int l = 0; l < D.L - 1; ++l) c->dMask[l] = cv.take<uint4>(rows_t);
  c->dZb[0] = cv.take<float>(rows_t * D.maxw);
  c->dZb[1] = cv.take<float>(rows_t * D.maxw);
  c->logits_d = cv.take<float>(2 * N);
  c->logits_g = cv.take<float>(N);
  c->dy = cv.take<float>(2 * N);
  c->hist = cv.take<uint32_t>(4 * (g.hist_bins + 2));
  // split-K partials: the largest wgrad of either network, or the head
  int64_t pf = (int64_t)head_blocks() * (D.maxw + 1);
  for (int l = 0; l < D.L - 1; ++l)
    pf = std::max<int64_t>(pf, (int64_t)wgrad_splits(D.sizes[l + 1], D.sizes[l], 2 * N) * D.sizes[l + 1] * D.sizes[l]);
  for (int l = 0; l < G.L; ++l)
    pf = std::max<int64_t>(pf, (int64_t)wgrad_splits(G.sizes[l + 1], G.sizes[l], k) * G.sizes[l + 1] * G.sizes[l]);
  pf = std::max<int64_t>(pf, (int64_t)kMaxSms * 128 * 128);  // tcgen05 wgrad: one partial per CTA
  c->part = cv.take<float>(pf);
  c->part_floats = pf;
  c->colpart = cv.take<float>(std::max<int64_t>((int64_t)std::max(296, kMaxSms) * std::max(128, std::max(D.maxw, G.maxw)),
                                                (int64_t)kMaxSms * 4 * 384));
  c->head_tmp = cv.take<float>(D.maxw + 1);
  c->dbpart = cv.take<float>((int64_t)kMaxSms * 128);
  c->tile_ctrs = cv.take<uint32_t>(sagips_ctx::kTileCtrs);
  if (c->cfg.disc_hidden == 128) {  // per-layer wgrad partials of the tcgen05 layer passes (reduced + Adam at the end)
    for (int l = 1; l + 1 < D.L; ++l) {
      c->lpart[l] = cv.take<float>((int64_t)kMaxSms * 128 * 128);
      c->ldb[l] = cv.take<float>((int64_t)kMaxSms * 128);
    }
  }
  c->loss_part = cv.take<double>(head_blocks());
  c->stats = cv.take<sagips_step_stats>(1);
  for (int b = 0; b < 2; ++b) c->hin[b] = cv.take<float>(k * g.noise_dim + 2 * N);  // host-input staging
  c->ws_bytes = cv.off;
}

}  // namespace sagips

using namespace sagips;

// ---------------------------------------------------------------- helpers
static sagips_status fail(sagips_ctx* c, sagips_status s, const char* fmt, ...) {
  if (c) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    c->err = buf;
  }
  return s;
}

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) return fail(ctx, SAGIPS_ERR_CUDA, "%s: %s (%s:%d)", #call,         \
                                       cudaGetErrorString(e_), __FILE__, __LINE__);           \
  } while (0)

static int tab_grid(const sagips_config& g) { return g.sampler_grid > 0 ? g.sampler_grid : 1024; }

static sagips_status validate(const sagips_config* g, std::string* why) {
  auto bad = [&](const char* m) { *why = m; return SAGIPS_ERR_CONFIG; };
  if (g->world < 1 || g->world > kMaxWorld) return bad("world must be in [1, 64]");
  if (g->rank < 0 || g->rank >= g->world) return bad("rank out of range");
  if (g->group_size < 1) return bad("group_size must be >= 1");
  if (g->outer_rma != 0 && g->outer_rma != 1) return bad("outer_rma must be 0 or 1");
  if (g->mode < SAGIPS_MODE_NONE || g->mode > SAGIPS_MODE_RMA_CHUNKED) return bad("unknown mode");
  if (g->mode == SAGIPS_MODE_RMA_CHUNKED && g->staleness != 0)
    return bad("RMA_CHUNKED reduces one common sum: staleness must be 0");
  if (g->staleness < 0 || g->staleness > 1) return bad("staleness must be 0 or 1");
  if (g->precision != SAGIPS_PREC_FP32 && g->precision != SAGIPS_PREC_BF16) return bad("unknown precision");
  if (g->noise_dim < 1 || g->gen_hidden < 1 || g->gen_depth < 1 || g->disc_depth < 1) return bad("model dims");
  if (g->gen_depth + 1 > kMaxLayers || g->disc_depth + 1 > kMaxLayers) return bad("too many layers");
  const int hd = g->disc_hidden;
  if (hd != 32 && hd != 64 && hd != 128 && hd != 256) return bad("disc_hidden must be 32, 64, 128 or 256");
  if (g->param_samples < 1 || g->events_per_sample < 1) return bad("k, m >= 1");
  const int64_t N = (int64_t)g->param_samples * g->events_per_sample;
  if (2 * N >= (1LL << 31)) return bad("2N must be < 2^31");
  if (g->reference_rows < 1 || g->reference_rows >= (1LL << 32)) return bad("reference_rows in [1, 2^32)");
  if (g->shard_rows < 1 || g->shard_rows >= (1LL << 32)) return bad("shard_rows in [1, 2^32)");
  if (g->sampler != SAGIPS_SAMPLER_QUADRATIC && g->sampler != SAGIPS_SAMPLER_TABULATED) return bad("unknown sampler");
  if (g->packet_biases != 0 && g->packet_biases != 1) return bad("packet_biases must be 0 or 1");
  if (g->sampler == SAGIPS_SAMPLER_TABULATED && g->sampler_grid != 0 && !tabulated_ok(g->sampler_grid))
    return bad("sampler_grid must be in [3, 2048]");
  for (int o = 0; o < 2; ++o)
    if (!(g->true_params[3 * o + 1] > 0.f) || !(g->true_params[3 * o + 2] > 0.f))
      return bad("true c1, c2 (tabulated: b, c) must be > 0 (softplus range)");
  if (g->sampler == SAGIPS_SAMPLER_TABULATED)
    for (int o = 0; o < 2; ++o)
      if (!(g->true_params[3 * o] > 0.f && g->true_params[3 * o] < 1.f)) return bad("true w must be in (0, 1)");
  if (g->hist_bins < 1 || g->hist_bins > 4096) return bad("hist_bins in [1, 4096]");
  if (!(g->leaky_slope >= 0.f && g->leaky_slope < 1.f)) return bad("leaky_slope must be in [0, 1) (R6)");
  if (g->disc_impl < SAGIPS_DISC_AUTO || g->disc_impl > SAGIPS_DISC_TCGEN05) return bad("unknown disc_impl");
  if (g->disc_impl == SAGIPS_DISC_TCGEN05 && hd != 128) return bad("tcgen05 layers need disc_hidden == 128");
  if (g->precision == SAGIPS_PREC_BF16 && (hd != 128 || g->disc_impl == SAGIPS_DISC_SIMT))
    return bad("BF16 precision runs on tcgen05 (disc_hidden == 128, disc_impl != SIMT)");
  for (int o = 0; o < 2; ++o)
    if (!(g->hist_hi[o] > g->hist_lo[o])) return bad("hist_hi must exceed hist_lo");
  return SAGIPS_OK;
}

static void setup_dims(sagips_ctx* c) {
  const sagips_config& g = c->cfg;
  c->G.build(g.noise_dim, g.gen_hidden, g.gen_depth, 6);   // Eq. 4: six parameters
  c->D.build(2, g.disc_hidden, g.disc_depth, 1);           // two observables -> one logit
  c->N = (int64_t)g.param_samples * g.events_per_sample;
}

extern "C" {

int32_t sagips_abi_version(void) { return SAGIPS_ABI_VERSION; }

sagips_status sagips_config_init(sagips_config* cfg, int32_t preset) {
  if (!cfg) return SAGIPS_ERR_INVALID_ARG;
  std::memset(cfg, 0, sizeof *cfg);
  cfg->world = 1; cfg->rank = 0; cfg->group_size = 1; cfg->outer_every = 0;
  cfg->mode = SAGIPS_MODE_NONE; cfg->staleness = 0; cfg->reduce_mean = 1;
  cfg->precision = SAGIPS_PREC_FP32;
  cfg->gen_lr = 1e-5f; cfg->disc_lr = 1e-4f; cfg->leaky_slope = 0.01f;
  cfg->adam_beta1 = 0.9f; cfg->adam_beta2 = 0.999f; cfg->adam_eps = 1e-8f;
  const float p[6] = {1.0f, 1.0f, 0.5f, 2.0f, 0.5f, 1.0f};
  std::memcpy(cfg->true_params, p, sizeof p);
  cfg->hist_bins = 64;
  cfg->hist_lo[0] = cfg->hist_lo[1] = 0.0f;
  cfg->hist_hi[0] = cfg->hist_hi[1] = 4.0f;
  cfg->seed = 1;
  cfg->exchange_timeout_ms = 10000;
  if (preset == SAGIPS_PRESET_DESK) {
    cfg->noise_dim = 8; cfg->gen_hidden = 64; cfg->gen_depth = 2; cfg->disc_hidden = 64; cfg->disc_depth = 2;
    cfg->param_samples = 64; cfg->events_per_sample = 16;
  } else if (preset == SAGIPS_PRESET_PAPER) {
    cfg->noise_dim = 6; cfg->gen_hidden = 128; cfg->gen_depth = 4; cfg->disc_hidden = 128; cfg->disc_depth = 4;
    cfg->param_samples = 1024; cfg->events_per_sample = 1024;
  } else {
    return SAGIPS_ERR_INVALID_ARG;
  }
  const int64_t N = (int64_t)cfg->param_samples * cfg->events_per_sample;
  cfg->reference_rows = 2 * N;  // R18: n_s = 50% of N_ref = N
  cfg->shard_rows = N;
  return SAGIPS_OK;
}

sagips_status sagips_workspace_size(const sagips_config* cfg, size_t* bytes) {
  if (!cfg || !bytes) return SAGIPS_ERR_INVALID_ARG;
  std::string why;
  sagips_status s = validate(cfg, &why);
  if (s != SAGIPS_OK) return s;
  sagips_ctx tmp;
  tmp.cfg = *cfg;
  setup_dims(&tmp);
  carve(&tmp, nullptr);
  *bytes = tmp.ws_bytes + 256;
  return SAGIPS_OK;
}

const char* sagips_last_error(const sagips_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

sagips_status sagips_create(const sagips_config* cfg, void* workspace, size_t workspace_bytes, void* stream,
                            sagips_ctx** out) {
  if (!cfg || !workspace || !out) return SAGIPS_ERR_INVALID_ARG;
  *out = nullptr;
  std::string why;
  sagips_status s = validate(cfg, &why);
  if (s != SAGIPS_OK) {
    fprintf(stderr, "sagips_create: %s\n", why.c_str());
    return s;
  }
  sagips_ctx* ctx = new sagips_ctx();
  ctx->cfg = *cfg;
  if (ctx->cfg.exchange_timeout_ms <= 0) ctx->cfg.exchange_timeout_ms = 10000;
  setup_dims(ctx);
  ctx->use_tc = ctx->cfg.disc_impl != SAGIPS_DISC_SIMT && ctx->cfg.disc_hidden == 128;
  char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(workspace) + 255) & ~uintptr_t(255));
  carve(ctx, base);
  if ((size_t)(base - (char*)workspace) + ctx->ws_bytes > workspace_bytes) {
    delete ctx;
    return SAGIPS_ERR_INVALID_ARG;
  }
  ctx->launch_base = launches_total();
  cudaGetDevice(&ctx->dev);
  cudaStream_t st = (cudaStream_t)stream;
  const sagips_config& g = ctx->cfg;
  auto bail = [&](sagips_status r) { *out = nullptr; return r; };
  // Kaiming-normal weights: G identical on every rank, D per rank
  const float a = g.leaky_slope;
  for (int l = 0; l < ctx->G.L; ++l) {
    const float std_ = std::sqrt(2.0f / ((1.0f + a * a) * ctx->G.sizes[l]));
    launch_normals(ctx->gW + ctx->G.w_off[l], (int64_t)ctx->G.sizes[l + 1] * ctx->G.sizes[l], std_, g.seed, l, 0,
                   kStreamInitG, st);
  }
  for (int l = 0; l < ctx->D.L; ++l) {
    const float std_ = std::sqrt(2.0f / ((1.0f + a * a) * ctx->D.sizes[l]));
    launch_normals(ctx->dW + ctx->D.w_off[l], (int64_t)ctx->D.sizes[l + 1] * ctx->D.sizes[l], std_, g.seed, l,
                   g.rank, kStreamInitD, st);
  }
  cudaError_t e = cudaSuccess;
  e = cudaMemsetAsync(ctx->gB, 0, sizeof(float) * ctx->G.nb, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(ctx->dB, 0, sizeof(float) * ctx->D.nb, st);
  for (float* p : {ctx->gmW, ctx->gvW, ctx->dmW, ctx->dvW})
    if (e == cudaSuccess) e = cudaMemsetAsync(p, 0, sizeof(float) * (p == ctx->gmW || p == ctx->gvW ? ctx->G.nw : ctx->D.nw), st);
  for (float* p : {ctx->gmB, ctx->gvB, ctx->dmB, ctx->dvB})
    if (e == cudaSuccess) e = cudaMemsetAsync(p, 0, sizeof(float) * (p == ctx->gmB || p == ctx->gvB ? ctx->G.nb : ctx->D.nb), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(ctx->stats, 0, sizeof(sagips_step_stats), st);
  // loop-closure reference and the rank's shard
  if (g.sampler == SAGIPS_SAMPLER_TABULATED) {
    // reference events from the tabulated sampler at the true (w, b, c) (R32):
    // raw_true = (logit w, log expm1 b, log expm1 c) in fp32, word 2e+o of the REF stream
    float rt[6];
    for (int o = 0; o < 2; ++o) {
      const double w = g.true_params[3 * o], b = g.true_params[3 * o + 1], cc = g.true_params[3 * o + 2];
      rt[3 * o] = (float)std::log(w / (1.0 - w));
      rt[3 * o + 1] = (float)(b > 20.0 ? b : std::log(std::expm1(b)));
      rt[3 * o + 2] = (float)(cc > 20.0 ? cc : std::log(std::expm1(cc)));
    }
    if (e == cudaSuccess) e = cudaMemcpy(ctx->draw, rt, sizeof rt, cudaMemcpyHostToDevice);  // scratch
    launch_sample_tabulated(ctx->draw, 1, (int)g.reference_rows, tab_grid(g), g.seed, 0, 0, kStreamRef, ctx->ref, st);
  } else {
    launch_reference(ctx->ref, g.reference_rows, g.true_params, g.seed, st);
  }
  launch_shard(ctx->ref, g.reference_rows, ctx->shard, g.shard_rows, g.seed, g.rank, st);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    fprintf(stderr, "sagips_create: %s\n", cudaGetErrorString(e));
    delete ctx;
    return bail(SAGIPS_ERR_CUDA);
  }
  *out = ctx;
  return SAGIPS_OK;
}

sagips_status sagips_destroy(sagips_ctx* ctx) {
  if (!ctx) return SAGIPS_ERR_INVALID_ARG;
  fused_trace_report();
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  if (ctx->cstream) cudaStreamDestroy(ctx->cstream);
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
    for (int b = 0; b < 2; ++b) {
      cudaEventDestroy(ctx->in_ready[b]);
      cudaEventDestroy(ctx->in_free[b]);
    }
  }
  exchange_destroy(ctx);
  for (auto& row : ctx->pev)
    for (auto& e : row)
      if (e) cudaEventDestroy(e);
  delete ctx;
  return SAGIPS_OK;
}

sagips_status sagips_sample_events(const float* c, int32_t k, int32_t m, uint64_t seed, uint64_t step, uint32_t rank,
                                   uint32_t stream_id, float* events, uint32_t* hist, int32_t bins, const float* lo,
                                   const float* hi, void* stream) {
  if (!c || !events || k < 1 || m < 1) return SAGIPS_ERR_INVALID_ARG;
  if (hist && (bins < 1 || !lo || !hi || !(hi[0] > lo[0]) || !(hi[1] > lo[1]))) return SAGIPS_ERR_INVALID_ARG;
  if ((int64_t)k * m >= (1LL << 31)) return SAGIPS_ERR_INVALID_ARG;
  launch_sample_events(c, k, m, seed, (uint32_t)step, rank, stream_id, events, hist, bins, lo, hi,
                       (cudaStream_t)stream);
  return cudaGetLastError() == cudaSuccess ? SAGIPS_OK : SAGIPS_ERR_CUDA;
}

sagips_status sagips_sample_tabulated(const float* raw, int32_t k, int32_t m, int32_t G, uint64_t seed,
                                      uint64_t step, uint32_t rank, uint32_t stream_id, float* events, void* stream) {
  if (!raw || !events || k < 1 || m < 1 || !tabulated_ok(G) || (int64_t)k * m >= (1LL << 31))
    return SAGIPS_ERR_INVALID_ARG;
  launch_sample_tabulated(raw, k, m, G, seed, (uint32_t)step, rank, stream_id, events, (cudaStream_t)stream);
  return cudaGetLastError() == cudaSuccess ? SAGIPS_OK : SAGIPS_ERR_CUDA;
}

sagips_status sagips_sample_tabulated_bwd(const float* raw, int32_t k, int32_t m, int32_t G, uint64_t seed,
                                          uint64_t step, uint32_t rank, uint32_t stream_id, const float* dy,
                                          float* draw, void* stream) {
  if (!raw || !dy || !draw || k < 1 || m < 1 || !tabulated_ok(G) || (int64_t)k * m >= (1LL << 31))
    return SAGIPS_ERR_INVALID_ARG;
  launch_sample_tabulated_bwd(raw, k, m, G, seed, (uint32_t)step, rank, stream_id, dy, draw, (cudaStream_t)stream);
  return cudaGetLastError() == cudaSuccess ? SAGIPS_OK : SAGIPS_ERR_CUDA;
}

sagips_status sagips_predict_params(sagips_ctx* ctx, const float* noise, int32_t k, float* c_out, void* stream) {
  if (!ctx || !noise || !c_out || k < 1 || k > ctx->cfg.param_samples) return SAGIPS_ERR_INVALID_ARG;
  if (!gen_fused_ok(ctx)) return SAGIPS_ERR_UNSUPPORTED;
  launch_gen_predict(ctx, noise, k, c_out, (cudaStream_t)stream);
  return cudaGetLastError() == cudaSuccess ? SAGIPS_OK : SAGIPS_ERR_CUDA;
}

sagips_status sagips_ensemble_stats(const float* preds, int32_t M, int32_t k, int32_t P, const double* p_true,
                                    double* out, void* stream) {
  if (!preds || !out || M < 1 || k < 1 || P < 1 || P > kEnsMaxParams) return SAGIPS_ERR_INVALID_ARG;
  const cudaStream_t st = (cudaStream_t)stream;
  double* d_out = nullptr;
  if (cudaMalloc(&d_out, sizeof(double) * 3 * P) != cudaSuccess) return SAGIPS_ERR_CUDA;
  const int rc = launch_ensemble_stats(preds, M, k, P, p_true, d_out, st);
  cudaError_t e = cudaMemcpyAsync(out, d_out, sizeof(double) * 3 * P, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(d_out);
  return (rc == 0 && e == cudaSuccess) ? SAGIPS_OK : SAGIPS_ERR_CUDA;
}

}  // extern "C"

// ---------------------------------------------------------------- the step
namespace sagips {

// A 128 -> 128 discriminator layer runs on the tensor cores (tcgen05) unless
// disc_impl == SIMT; FP32 precision uses the bf16x3 split (fp32-class).
static bool tc_layer(const sagips_ctx* c, int l) {
  return c->use_tc && c->D.sizes[l] == 128 && c->D.sizes[l + 1] == 128;
}
static bool tc_split(const sagips_ctx* c) { return c->cfg.precision == SAGIPS_PREC_FP32; }

// Hidden layers of the discriminator on `rows` rows of X -> dAct[0..L-2].
static void disc_hidden_forward(sagips_ctx* c, const float* X, int rows, cudaStream_t st) {
  const auto& D = c->D;
  const float* in = X;
  for (int l = 0; l < D.L - 1; ++l) {
    if (tc_layer(c, l)) {
      launch_tc_rows(tc_split(c), false, in, c->dW + D.w_off[l], c->dAct[l], rows, EPI_BIAS_ACT, c->dB + D.b_off[l],
                     nullptr, c->cfg.leaky_slope, st);
    } else {
      Epi ep{EPI_BIAS_ACT, c->dB + D.b_off[l], 1, c->cfg.leaky_slope, nullptr, 0};
      launch_gemm(false, true, rows, D.sizes[l + 1], D.sizes[l], in, D.sizes[l], c->dW + D.w_off[l], D.sizes[l],
                  c->dAct[l], D.sizes[l + 1], ep, 1, 0, st);
    }
    in = c->dAct[l];
  }
}

// wgrad + bias grad of one layer: dW = dZ^T Hin (K = rows), db = colsum(dZ).
static void layer_wgrad(sagips_ctx* c, const float* dZ, const float* Hin, int rows, int out, int in, float* dW,
                        float* db, cudaStream_t st) {
  const int S = wgrad_splits(out, in, rows);
  Epi ep{EPI_STORE, nullptr, 0, 0.f, nullptr, 0};
  launch_gemm(true, false, out, in, rows, dZ, out, Hin, in, c->part, in, ep, S, (int64_t)out * in, st);
  launch_reduce_parts(c->part, S, (int64_t)out * in, dW, 1.0f, st);
  const int S2 = (int)std::min<int64_t>(296, std::max(1, rows / 256));
  launch_colsum(dZ, rows, out, out, S2, c->colpart, st);
  launch_reduce_parts(c->colpart, S2, out, db, 1.0f, st);
}

static void disc_layer_wgrad(sagips_ctx* c, int l, const float* dZ, const float* Hin, int rows, cudaStream_t st) {
  const auto& D = c->D;
  if (tc_layer(c, l)) {
    launch_tc_wgrad(tc_split(c), dZ, Hin, rows, c->part, c->colpart, st);
    launch_reduce_parts(c->part, tc_wgrad_grid(), 128 * 128, c->d_dW + D.w_off[l], 1.0f, st);
    launch_reduce_parts(c->colpart, tc_wgrad_grid(), 128, c->d_dB + D.b_off[l], 1.0f, st);
  } else {
    layer_wgrad(c, dZ, Hin, rows, D.sizes[l + 1], D.sizes[l], c->d_dW + D.w_off[l], c->d_dB + D.b_off[l], st);
  }
}

// dZ_{l-1} = (dZ_l W_l) * LeakyReLU'(H_{l-1})
static void disc_layer_dgrad(sagips_ctx* c, int l, const float* dZ, float* out_dZ, int rows, cudaStream_t st) {
  const auto& D = c->D;
  const int out = D.sizes[l + 1], in = D.sizes[l];
  if (tc_layer(c, l)) {
    launch_tc_rows(tc_split(c), true, dZ, c->dW + D.w_off[l], out_dZ, rows, EPI_ACT_GRAD, nullptr, c->dAct[l - 1],
                   c->cfg.leaky_slope, st);
  } else {
    Epi ep{EPI_ACT_GRAD, nullptr, 0, c->cfg.leaky_slope, c->dAct[l - 1], in};
    launch_gemm(false, false, rows, in, out, dZ, out, c->dW + D.w_off[l], in, out_dZ, in, ep, 1, 0, st);
  }
}

// ---- warp-specialised tcgen05 layer passes (k_tc_layers.cu), depth >= 3.
// Layer 0 is recomputed from X inside the first pass; the head + BCE is the
// epilogue of the last hidden layer; dgrad and wgrad share one pass.
static bool use_layers_v2(const sagips_ctx* c) { return c->use_tc && c->cfg.disc_depth >= 3; }

// plane tiles of a whole tensor (per-layer kernels)
static Ring whole(void* base, uint4* mask = nullptr) {
  Ring r;
  r.base = reinterpret_cast<uint8_t*>(base);
  r.mask = mask;
  return r;
}

// dynamic tile-schedule counters: one per launch of a step, zeroed at the
// start of each D / G step (SAGIPS_DYN=0 disables the dynamic schedule)
static uint32_t* next_tile_ctr(sagips_ctx* c) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("SAGIPS_DYN");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  if (!env || c->tile_ctr_next >= sagips_ctx::kTileCtrs) return nullptr;
  return c->tile_ctrs + c->tile_ctr_next++;
}
static void reset_tile_ctrs(sagips_ctx* c, cudaStream_t st) {
  cudaMemsetAsync(c->tile_ctrs, 0, sizeof(uint32_t) * sagips_ctx::kTileCtrs, st);
  c->tile_ctr_next = 0;
}

// The first forward layer's 4 producer warps make all 128 H_1 rows of a tile
// (measured: D 0.379 vs 0.401 ms, G 0.153 vs 0.187 ms at C2, r01 v11);
// SAGIPS_FIRST_HELP=1: the epilogue warps make rows 64-127 after each tile
static int first_help() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SAGIPS_FIRST_HELP");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v;
}

// SAGIPS_H1_STORE=1: the D forward's first layer stores the H_1 hi plane and
// the layer-1 backward bulk-loads it; default: the backward's producer warps
// recompute it from X (512 B/row less HBM traffic)
static bool h1_store() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SAGIPS_H1_STORE");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

static bool use_fused(const sagips_ctx* c);
static bool tc_split(const sagips_ctx* c);
static bool h1_store();
// the fused D step passes G_4 as dz + sign bits (kGenG; the default, both
// precisions; SAGIPS_GEN_G=0 writes the planes instead)
static bool gen_g(const sagips_ctx* c) {
  const char* e = getenv("SAGIPS_GEN_G");
  return !(e && e[0] == '0') && use_fused(c) && !h1_store();
}

static void disc_forward_v2(sagips_ctx* c, const float* X, int64_t rows, int64_t n_real, float label_rest,
                            float scale, float* logits, bool want_grads, cudaStream_t st) {
  const int kc = want_grads ? 0 : 6;  // kernel-timing classes
  const bool split = tc_split(c);
  const auto& D = c->D;
  const int Lh = D.L - 1;
  if (want_grads && use_fused(c) && !h1_store()) {
    // the D step's forward in one kernel (k_fused.cu): H_2 / H_3 hi planes and
    // masks and the G_4 planes for the per-layer backward passes
    DFwdArgs f{};
    f.X = reinterpret_cast<const float2*>(X);
    f.rows = rows;
    f.n_real = n_real;
    f.label_rest = label_rest;
    f.scale = scale;
    for (int l = 0; l < 4; ++l) {
      f.W[l] = c->dW + D.w_off[l];
      f.b[l] = c->dB + D.b_off[l];
    }
    f.w4 = c->dW + D.w_off[4];
    f.b4 = c->dB + D.b_off[4];
    f.alpha = c->cfg.leaky_slope;
    f.logits = logits;
    f.loss_part = c->loss_part;
    f.part_head = c->part;
    f.h2 = reinterpret_cast<uint8_t*>(c->dAct[1]);
    f.m2 = c->dMask[1];
    f.h3 = reinterpret_cast<uint8_t*>(c->dAct[2]);
    f.m3 = c->dMask[2];
    // fp32-class: dz and the Z_4 sign bits (in the otherwise
    // unused H_4 buffers) replace the G_4 planes and the next pass
    // regenerates them (SAGIPS_GEN_G=0: the planes)
    f.g4 = gen_g(c) ? nullptr : reinterpret_cast<uint8_t*>(c->dZb[0]);
    f.dz = c->dAct[3];
    f.m4 = c->dMask[3];
    f.trace = fused_trace_buffer();
    kernel_begin(c, 13, st);
    launch_dfwd(split, f, st);
    kernel_end(c, st);
    return;
  }
  FwdLaunch f;  // H_2 = LeakyReLU(H_1 W_1^T + b_1), H_1 recomputed from X
  f.X = X; f.W0 = c->dW + D.w_off[0]; f.b0 = c->dB + D.b_off[0]; f.first_help = first_help();
  f.W = c->dW + D.w_off[1]; f.bias = c->dB + D.b_off[1]; f.out = whole(c->dAct[1], c->dMask[1]);
  f.rows = rows; f.alpha = c->cfg.leaky_slope;
  if (want_grads && split && h1_store()) f.h1 = whole(c->dAct[0]);  // H_1 hi plane for the layer-1 wgrad
  kernel_begin(c, kc + 0, st);
  launch_tc_fwd(split, FWD_FIRST, f, st);
  kernel_end(c, st);
  for (int l = 2; l <= Lh - 2; ++l) {  // H_{l+1} = LeakyReLU(H_l W_l^T + b_l)
    FwdLaunch m;
    m.in = whole(c->dAct[l - 1]); m.W = c->dW + D.w_off[l]; m.bias = c->dB + D.b_off[l];
    m.out = whole(c->dAct[l], c->dMask[l]);
    m.rows = rows; m.alpha = c->cfg.leaky_slope;
    m.tile_ctr = next_tile_ctr(c);
    kernel_begin(c, kc + 1, st);
    launch_tc_fwd(split, FWD_MID, m, st);
    kernel_end(c, st);
  }
  FwdLaunch h;  // last hidden layer + head + BCE -> G_{Lh} planes
  h.in = whole(c->dAct[Lh - 2]); h.W = c->dW + D.w_off[Lh - 1]; h.bias = c->dB + D.b_off[Lh - 1];
  h.rows = rows; h.alpha = c->cfg.leaky_slope;
  h.w_head = c->dW + D.w_off[Lh]; h.b_head = c->dB + D.b_off[Lh];
  h.n_real = n_real; h.label_rest = label_rest; h.scale = scale;
  h.logits = logits; h.out = whole(c->dZb[0]); h.part_head = c->part;
  h.loss_part = c->loss_part; h.want_wgrad = want_grads ? 1 : 0;
  kernel_begin(c, kc + 2, st);
  launch_tc_fwd(split, FWD_HEAD, h, st);
  kernel_end(c, st);
}

// All discriminator gradients of a tcgen05 D step from their per-CTA partials
// (head [hparts][129], hidden layer l: lpart/ldb [nparts[l]], layer 0
// colpart [l0parts][384]) -> d_dW / d_dB, then Adam(D): one launch.
// loss_scale > 0: the D loss partials (c->loss_part, hparts of them) are
// finished by the reduction's extra block
static void disc_reduce_adam(sagips_ctx* c, int hparts, const int* nparts, int l0parts, cudaStream_t st,
                             double loss_scale = 0.0) {
  const auto& D = c->D;
  const auto& g = c->cfg;
  const int Lh = D.L - 1;
  RedAdamArgs A;
  auto seg = [&](const float* part, int np, int64_t ld, int n, bool w, int l) {
    RedSeg& s = A.seg[A.nseg++];
    const int64_t off = w ? D.w_off[l] : D.b_off[l];
    s.part = part; s.nparts = np; s.ld = ld; s.n = n;
    s.g = (w ? c->d_dW : c->d_dB) + off;
    s.p = (w ? c->dW : c->dB) + off;
    s.m = (w ? c->dmW : c->dmB) + off;
    s.v = (w ? c->dvW : c->dvB) + off;
  };
  seg(c->part, hparts, 129, 128, true, Lh);        // head weights
  seg(c->part + 128, hparts, 129, 1, false, Lh);   // head bias
  for (int l = Lh - 1; l >= 1; --l) {
    seg(c->lpart[l], nparts[l], 128 * 128, 128 * 128, true, l);
    seg(c->ldb[l], nparts[l], 128, 128, false, l);
  }
  seg(c->colpart, l0parts, 384, 256, true, 0);     // dW_0 [128][2]
  seg(c->colpart + 256, l0parts, 384, 128, false, 0);
  if (loss_scale > 0.0) {
    A.loss_part = c->loss_part;
    A.loss_nparts = hparts;
    A.loss_scale = loss_scale;
    A.loss_out = &c->stats->loss_d;
    A.nonfinite = &c->stats->nonfinite;
  }
  c->d_tau += 1;
  launch_reduce_adam(A, g.disc_lr, c->d_tau, g.adam_beta1, g.adam_beta2, g.adam_eps, st);
  c->d_adam_done = true;
}

static void disc_step_v2(sagips_ctx* c, cudaStream_t st) {
  const auto& D = c->D;
  const int64_t N = c->N, rows = 2 * N;
  const int Lh = D.L - 1;
  const bool split = tc_split(c);
  const int grid = tc_layers_grid(rows);
  reset_tile_ctrs(c, st);
  disc_forward_v2(c, c->X, rows, N, 0.0f, 1.0f / (float)rows, c->logits_d, true, st);
  // (the loss partials wait in loss_part: k_reduce_adam's extra block finishes L_D)
  int cur = 0;
  int nparts[kMaxLayers] = {};
  for (int l = Lh - 1; l >= 1; --l) {
    BwdLaunch b;
    b.g = whole(c->dZb[cur]); b.W = c->dW + D.w_off[l]; b.rows = rows;
    b.alpha = c->cfg.leaky_slope; b.part = c->lpart[l]; b.part_db = c->ldb[l];
    if (l == Lh - 1 && gen_g(c)) {  // G_4 from k_dfwd's dz + sign bits
      b.gen_dz = c->dAct[3];
      b.gen_mask = c->dMask[3];
      b.gen_w = c->dW + D.w_off[Lh];
    }
    nparts[l] = grid;
    if (l == 1) {
      b.X = c->X; b.W0 = c->dW + D.w_off[0]; b.b0 = c->dB + D.b_off[0]; b.part_l0 = c->colpart;
      if (split && h1_store()) b.h = whole(c->dAct[0]);  // H_1 hi plane stored by the forward first layer
    } else {
      b.h = whole(c->dAct[l - 1], c->dMask[l - 1]);
      b.gout = whole(c->dZb[cur ^ 1]);
    }
    kernel_begin(c, l == Lh - 1 ? 3 : l == 1 ? 5 : 4, st);
    launch_tc_bwd(split, l == 1, true, b, st);
    kernel_end(c, st);
    cur ^= 1;
  }
  disc_reduce_adam(c, grid, nparts, grid, st, 1.0 / rows);
}

// the fused G step (k_fused.cu): paper widths, depth 4; SAGIPS_FUSED=0 keeps the per-layer kernels
static bool use_fused(const sagips_ctx* c) {
  const char* e = getenv("SAGIPS_FUSED");
  const bool env = !(e && e[0] == '0');
  return env && c->use_tc && c->cfg.disc_depth == 4 && c->cfg.disc_hidden == 128;
}

static void gen_loss_v2(sagips_ctx* c, cudaStream_t st) {
  const auto& D = c->D;
  const int64_t N = c->N;
  const int Lh = D.L - 1;
  const bool split = tc_split(c);
  const float* Y = c->X + 2 * N;  // fake rows
  if (use_fused(c)) {
    GStepArgs a{};
    a.Y = reinterpret_cast<const float2*>(Y);
    a.rows = N;
    for (int l = 0; l < 4; ++l) {
      a.W[l] = c->dW + D.w_off[l];
      a.b[l] = c->dB + D.b_off[l];
    }
    a.w4 = c->dW + D.w_off[4];
    a.b4 = c->dB + D.b_off[4];
    a.alpha = c->cfg.leaky_slope;
    a.scale = 1.0f / (float)N;
    a.logits = c->logits_g;
    a.loss_part = c->loss_part;
    a.dy = reinterpret_cast<float2*>(c->dy);
    a.trace = fused_trace_buffer();
    kernel_begin(c, 12, st);
    launch_gstep(split, a, st);
    kernel_end(c, st);
    if (c->cfg.sampler == SAGIPS_SAMPLER_TABULATED) {
      launch_finish_loss(c->loss_part, fused_grid(N), 1.0 / N, &c->stats->loss_g, &c->stats->nonfinite, st);
    } else {  // finished by k_sample_bwd's extra block (the next launch)
      c->loss_g_defer = fused_grid(N);
      c->loss_g_scale = 1.0 / (double)N;
    }
    return;
  }
  reset_tile_ctrs(c, st);
  disc_forward_v2(c, Y, N, 0, 1.0f, 1.0f / (float)N, c->logits_g, false, st);
  launch_finish_loss(c->loss_part, tc_layers_grid(N), 1.0 / N, &c->stats->loss_g, &c->stats->nonfinite, st);
  int cur = 0;
  for (int l = Lh - 1; l >= 1; --l) {
    BwdLaunch b;
    b.g = whole(c->dZb[cur]); b.W = c->dW + D.w_off[l]; b.rows = N;
    b.alpha = c->cfg.leaky_slope;
    b.tile_ctr = next_tile_ctr(c);
    if (l == 1) {
      b.X = Y; b.W0 = c->dW + D.w_off[0]; b.b0 = c->dB + D.b_off[0]; b.dy = c->dy;
    } else {
      b.h = whole(nullptr, c->dMask[l - 1]); b.gout = whole(c->dZb[cur ^ 1]);
    }
    kernel_begin(c, l == Lh - 1 ? 9 : l == 1 ? 11 : 10, st);
    launch_tc_bwd(split, l == 1, false, b, st);
    kernel_end(c, st);
    cur ^= 1;
  }
}

static void disc_step(sagips_ctx* c, cudaStream_t st) {
  if (use_layers_v2(c)) {
    disc_step_v2(c, st);
    return;
  }
  const auto& D = c->D;
  const int N = (int)c->N;
  const int rows = 2 * N;
  const float a = c->cfg.leaky_slope;
  const int Lh = D.L - 1;  // index of the head layer
  const int hd = D.sizes[Lh];
  disc_hidden_forward(c, c->X, rows, st);
  // head: logits, BCE (labels: real rows 1, fake rows 0; mean over 2N), dz
  launch_head(c->dAct[Lh - 1], rows, hd, c->dW + D.w_off[Lh], c->dB + D.b_off[Lh], N, 0.0f, 1.0f / (float)rows, a,
              c->logits_d, c->dZb[0], c->part, c->loss_part, true, st);
  launch_reduce_parts(c->part, head_blocks(), hd + 1, c->head_tmp, 1.0f, st);
  cudaMemcpyAsync(c->d_dW + D.w_off[Lh], c->head_tmp, sizeof(float) * hd, cudaMemcpyDeviceToDevice, st);
  cudaMemcpyAsync(c->d_dB + D.b_off[Lh], c->head_tmp + hd, sizeof(float), cudaMemcpyDeviceToDevice, st);
  launch_finish_loss(c->loss_part, head_blocks(), 1.0 / rows, &c->stats->loss_d, &c->stats->nonfinite, st);
  int cur = 0;
  for (int l = Lh - 1; l >= 0; --l) {
    const float* Hin = (l == 0) ? c->X : c->dAct[l - 1];
    disc_layer_wgrad(c, l, c->dZb[cur], Hin, rows, st);
    if (l > 0) {
      disc_layer_dgrad(c, l, c->dZb[cur], c->dZb[cur ^ 1], rows, st);
      cur ^= 1;
    }
  }
}

static void gen_loss_through_disc(sagips_ctx* c, cudaStream_t st) {
  if (use_layers_v2(c)) {
    gen_loss_v2(c, st);
    return;
  }
  const auto& D = c->D;
  const int N = (int)c->N;
  const float a = c->cfg.leaky_slope;
  const int Lh = D.L - 1;
  const int hd = D.sizes[Lh];
  const float* Y = c->X + 2 * (int64_t)N;  // fake rows
  disc_hidden_forward(c, Y, N, st);
  // non-saturating generator loss: label 1 on fake rows, mean over N
  launch_head(c->dAct[Lh - 1], N, hd, c->dW + D.w_off[Lh], c->dB + D.b_off[Lh], 0, 1.0f, 1.0f / (float)N, a,
              c->logits_g, c->dZb[0], c->part, c->loss_part, false, st);
  launch_finish_loss(c->loss_part, head_blocks(), 1.0 / N, &c->stats->loss_g, &c->stats->nonfinite, st);
  int cur = 0;
  for (int l = Lh - 1; l >= 0; --l) {
    const int out = D.sizes[l + 1], in = D.sizes[l];
    if (l > 0) {
      disc_layer_dgrad(c, l, c->dZb[cur], c->dZb[cur ^ 1], N, st);
      cur ^= 1;
    } else {
      Epi ep{EPI_STORE, nullptr, 0, 0.f, nullptr, 0};
      launch_gemm(false, false, N, in, out, c->dZb[cur], out, c->dW + D.w_off[0], in, c->dy, in, ep, 1, 0, st);
    }
  }
}

static void adam_disc(sagips_ctx* c, cudaStream_t st) {
  const auto& g = c->cfg;
  c->d_tau += 1;
  launch_adam(c->dW, c->d_dW, c->dmW, c->dvW, c->D.nw, g.disc_lr, c->d_tau, g.adam_beta1, g.adam_beta2, g.adam_eps, st);
  launch_adam(c->dB, c->d_dB, c->dmB, c->dvB, c->D.nb, g.disc_lr, c->d_tau, g.adam_beta1, g.adam_beta2, g.adam_eps, st);
}

GenAdam gen_adam_args(sagips_ctx* c) {
  const auto& g = c->cfg;
  c->g_tau += 1;
  // bias corrections in double on the host, as launch_adam
  const double bc1 = 1.0 - std::pow((double)g.adam_beta1, (double)c->g_tau);
  const double bc2 = 1.0 - std::pow((double)g.adam_beta2, (double)c->g_tau);
  GenAdam a{};
  a.pw = c->gW; a.mw = c->gmW; a.vw = c->gvW;
  a.pb = c->gB; a.mb = c->gmB; a.vb = c->gvB;
  a.gb_local = (g.packet_biases && g.world > 1) ? nullptr : c->g_dB;
  a.nw = c->G.nw;
  a.nb = c->G.nb;
  a.step_size = (float)((double)g.gen_lr / bc1);
  a.bc2_sqrt = (float)std::sqrt(bc2);
  a.b1 = g.adam_beta1;
  a.b2 = g.adam_beta2;
  a.eps = g.adam_eps;
  return a;
}

void adam_gen(sagips_ctx* c, cudaStream_t st) {
  const auto& g = c->cfg;
  c->g_tau += 1;
  launch_adam(c->gW, c->reduced, c->gmW, c->gvW, c->G.nw, g.gen_lr, c->g_tau, g.adam_beta1, g.adam_beta2, g.adam_eps, st);
  // biases: the local gradients, or the reduced ones with the fused packet
  const float* gb = (g.packet_biases && g.world > 1) ? c->reduced + c->G.nw : c->g_dB;
  launch_adam(c->gB, gb, c->gmB, c->gvB, c->G.nb, g.gen_lr, c->g_tau, g.adam_beta1, g.adam_beta2, g.adam_eps, st);
}

// Steps a1..a11: everything up to and including the packet.
static void local_step(sagips_ctx* c, uint64_t t, cudaStream_t st) {
  const sagips_config& g = c->cfg;
  const auto& G = c->G;
  const int k = g.param_samples, m = g.events_per_sample;
  const float a = g.leaky_slope;
  const uint32_t step = (uint32_t)t;
  mark(c, 0, st);
  // a1 noise ~ N(0,1) (or the caller's, sagips_train_step_host); with the
  // fused generator the forward kernel draws it itself
  const bool fused_gen = gen_fused_ok(c);
  if (c->in_noise)
    cudaMemcpyAsync(c->noise, c->in_noise, sizeof(float) * k * g.noise_dim, cudaMemcpyDeviceToDevice, st);
  else if (!fused_gen)
    launch_normals(c->noise, (int64_t)k * g.noise_dim, 1.0f, g.seed, step, g.rank, kStreamNoise, st);
  // a2 generator forward (hidden LeakyReLU, linear output) + a3 constrain
  const bool tab = g.sampler == SAGIPS_SAMPLER_TABULATED;
  // the real rows come from the resident shard: prefetch it into L2 and zero
  // the histograms inside the generator forward (the step's sampler follows)
  const bool boot = !c->in_real;
  if (fused_gen) {
    launch_gen_fwd(c, st, boot ? c->shard : nullptr, boot ? 8 * g.shard_rows : 0, boot ? c->hist : nullptr,
                   boot ? 4 * (g.hist_bins + 2) : 0, c->in_noise ? nullptr : &step);
  } else {
    const float* in = c->noise;
    for (int l = 0; l < G.L; ++l) {
      Epi ep{EPI_BIAS_ACT, c->gB + G.b_off[l], l < G.L - 1, a, nullptr, 0};
      launch_gemm(false, true, k, G.sizes[l + 1], G.sizes[l], in, G.sizes[l], c->gW + G.w_off[l], G.sizes[l],
                  c->gAct[l], G.sizes[l + 1], ep, 1, 0, st);
      in = c->gAct[l];
    }
    launch_constrain(c->gAct[G.L - 1], c->cbuf, k, st, g.sampler == SAGIPS_SAMPLER_TABULATED);
  }
  const float* raw = c->gAct[G.L - 1];
  // a4-a6 fused sampler + bootstrap + histograms (tabulated: the bootstrap
  // pass draws the real rows, the tabulated sampler the fake rows N..2N-1)
  mark(c, 1, st);
  if (c->in_real) {
    // the caller's real batch (rows 0..N-1) replaces the bootstrap (a5); the
    // fake rows and their histogram as usual, the real histogram is zero
    cudaMemcpyAsync(c->X, c->in_real, sizeof(float) * 2 * (int64_t)k * m, cudaMemcpyDeviceToDevice, st);
    cudaMemsetAsync(c->hist, 0, sizeof(uint32_t) * 4 * (g.hist_bins + 2), st);
    if (!tab)
      launch_sample_events(c->cbuf, k, m, g.seed, step, g.rank, kStreamFake, c->X + 2 * (int64_t)k * m,
                           c->hist + 2 * (g.hist_bins + 2), g.hist_bins, g.hist_lo, g.hist_hi, st);
  } else {
    launch_sample_step(c->cbuf, k, m, c->shard, g.shard_rows, g.seed, step, g.rank, c->X, c->real_idx, c->hist,
                       g.hist_bins, g.hist_lo, g.hist_hi, st, !tab, fused_gen);
  }
  if (tab)
    launch_sample_tabulated(raw, k, m, tab_grid(g), g.seed, step, g.rank, kStreamFake,
                            c->X + 2 * (int64_t)k * m, st, c->hist ? c->hist + 2 * (g.hist_bins + 2) : nullptr,
                            g.hist_bins, g.hist_lo, g.hist_hi);
  mark(c, 2, st);
  // a7 discriminator step + Adam(D) ; a8 generator loss through the updated D
  disc_step(c, st);
  if (c->d_adam_done) c->d_adam_done = false;  // applied by the fused gradient reduction
  else adam_disc(c, st);
  mark(c, 3, st);
  gen_loss_through_disc(c, st);
  mark(c, 4, st);
  // a9 sampler backward
  if (tab) launch_sample_tabulated_bwd(raw, k, m, tab_grid(g), g.seed, step, g.rank, kStreamFake, c->dy, c->draw, st);
  else {
    LossFinish lf;
    if (c->loss_g_defer) {
      lf.loss_part = c->loss_part;
      lf.nparts = c->loss_g_defer;
      lf.scale = c->loss_g_scale;
      lf.out = &c->stats->loss_g;
      lf.nonfinite = &c->stats->nonfinite;
    }
    launch_sample_bwd(c->dy, raw, k, m, g.seed, step, g.rank, c->draw, st, lf);
  }
  c->loss_g_defer = 0;
  mark(c, 5, st);
  // a10 generator backward (the output layer is linear: dZ_L = draw);
  // a11 the weight gradients land in g_dW, which *is* the packet layout
  if (fused_gen) {
    launch_gen_bwd(c, st);
    mark(c, 6, st);
    return;
  }
  const float* cur = c->draw;
  int buf = 0;
  for (int l = G.L - 1; l >= 0; --l) {
    const float* Hin = (l == 0) ? c->noise : c->gAct[l - 1];
    const int out = G.sizes[l + 1], inn = G.sizes[l];
    layer_wgrad(c, cur, Hin, k, out, inn, c->g_dW + G.w_off[l], c->g_dB + G.b_off[l], st);
    if (l > 0) {
      Epi ep{EPI_ACT_GRAD, nullptr, 0, a, c->gAct[l - 1], inn};
      launch_gemm(false, false, k, inn, out, cur, out, c->gW + G.w_off[l], inn, c->gdZ[buf], inn, ep, 1, 0, st);
      cur = c->gdZ[buf];
      buf ^= 1;
    }
  }
  mark(c, 6, st);
}

}  // namespace sagips

extern "C" {

// the step after validation: a1-a11, then push / pull (eager, or inside a capture)
static sagips_status step_body(sagips_ctx* ctx, uint64_t step, uint32_t flags, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (timing_on(ctx)) {
    if (!ctx->pev[0][0])
      for (auto& row : ctx->pev)
        for (auto& e : row) CK(cudaEventCreate(&e));
    ctx->pslot = (int)(ctx->timed_steps % sagips_ctx::kTimingRing);
    ctx->kcount[ctx->pslot] = 0;
  }
  local_step(ctx, step, st);
  CK(cudaGetLastError());
  ctx->have_step = true;
  ctx->last_step = step;
  ctx->pushed = false;
  ctx->local_done_step = step;
  if (flags & SAGIPS_STEP_LOCAL_ONLY) {
    mark(ctx, 7, st);
    if (timing_on(ctx)) ctx->timed_steps++;
    return SAGIPS_OK;
  }
  sagips_status s = sagips_push_generator_grad(ctx, step, stream);
  if (s != SAGIPS_OK) return s;
  if (flags & SAGIPS_STEP_NO_ADAM_G) {
    ctx->skip_adam_once = true;
  }
  return sagips_pull_generator_grad(ctx, step, stream);
}

sagips_status sagips_train_step(sagips_ctx* ctx, uint64_t step, uint32_t flags, void* stream) {
  if (!ctx) return SAGIPS_ERR_INVALID_ARG;
  if (ctx->have_step && step != ctx->last_step + 1)
    return fail(ctx, SAGIPS_ERR_STATE, "step %llu is not the next step (%llu)", (unsigned long long)step,
                (unsigned long long)(ctx->last_step + 1));
  if (!ctx->have_step && step != 0 && ctx->cfg.world > 1 && ctx->cfg.mode != SAGIPS_MODE_NONE && ctx->cfg.staleness > 0)
    return fail(ctx, SAGIPS_ERR_STATE, "the first exchanging step with staleness 1 must be step 0");
  {
    const sagips_status xs = exchange_poll(ctx);
    if (xs != SAGIPS_OK) return xs;
  }
  // CUDA graph: capture this step's launches and replay them as one graph
  // launch (the first step runs eagerly: lazy set-up, kernel attributes);
  // an executable graph is updated in place while the topology is unchanged
  // (host-input steps too: their staged inputs are copied into place by
  // memcpy nodes, whose source slot alternates -- an in-place update)
  const bool graph = (flags & SAGIPS_STEP_GRAPH) && ctx->have_step && exchange_graph_ok(ctx) &&
                     !exchange_outer_step(ctx, step);
  flags &= ~SAGIPS_STEP_GRAPH;
  if (!graph) return step_body(ctx, step, flags, stream);
  // captured on a library-owned stream (the caller's may be the legacy
  // default stream, which cannot be captured); replayed on the caller's
  if (!ctx->cstream) CK(cudaStreamCreateWithFlags(&ctx->cstream, cudaStreamNonBlocking));
  cudaStream_t cs = ctx->cstream;
  CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  ctx->capturing = true;
  sagips_status s = step_body(ctx, step, flags, cs);
  if (s == SAGIPS_OK && !(flags & SAGIPS_STEP_LOCAL_ONLY)) s = exchange_join(ctx, cs);
  ctx->capturing = false;
  cudaGraph_t g = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(cs, &g);
  cudaStream_t st = (cudaStream_t)stream;
  if (s != SAGIPS_OK) {
    if (g) cudaGraphDestroy(g);
    return s;
  }
  if (ec != cudaSuccess) return fail(ctx, SAGIPS_ERR_CUDA, "graph capture: %s", cudaGetErrorString(ec));
  if (ctx->gexec) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(ctx->gexec, g, &info) != cudaSuccess) {
      cudaGetLastError();
      cudaGraphExecDestroy(ctx->gexec);
      ctx->gexec = nullptr;
    }
  }
  if (!ctx->gexec) {
    const cudaError_t ei = cudaGraphInstantiate(&ctx->gexec, g, 0);
    if (ei != cudaSuccess) {
      cudaGraphDestroy(g);
      ctx->gexec = nullptr;
      return fail(ctx, SAGIPS_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(ei));
    }
    ctx->graph_instantiations++;
  }
  cudaGraphDestroy(g);
  CK(cudaGraphLaunch(ctx->gexec, st));
  ctx->graph_launches++;
  return SAGIPS_OK;
}

sagips_status sagips_train_step_host(sagips_ctx* ctx, uint64_t step, uint32_t flags, const float* host_noise,
                                     const float* host_real, sagips_step_stats* host_stats, void* stream) {
  if (!ctx) return SAGIPS_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  if (host_noise || host_real) {
    // copy_stream: H2D into staging slot b once the step that used b last
    // has copied it into place (in_free[b]); the step waits for in_ready[b]
    if (!ctx->copy_stream) {
      CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
      for (int b = 0; b < 2; ++b) {
        CK(cudaEventCreateWithFlags(&ctx->in_ready[b], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->in_free[b], cudaEventDisableTiming));
      }
    }
    const int b = (int)(step & 1);
    const int64_t nz = (int64_t)ctx->cfg.param_samples * ctx->cfg.noise_dim;
    if (ctx->in_free_recorded[b]) CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->in_free[b], 0));
    if (host_noise)
      CK(cudaMemcpyAsync(ctx->hin[b], host_noise, sizeof(float) * nz, cudaMemcpyHostToDevice, ctx->copy_stream));
    if (host_real)
      CK(cudaMemcpyAsync(ctx->hin[b] + nz, host_real, sizeof(float) * 2 * ctx->N, cudaMemcpyHostToDevice,
                         ctx->copy_stream));
    CK(cudaEventRecord(ctx->in_ready[b], ctx->copy_stream));
    CK(cudaStreamWaitEvent(st, ctx->in_ready[b], 0));
    ctx->in_noise = host_noise ? ctx->hin[b] : nullptr;
    ctx->in_real = host_real ? ctx->hin[b] + nz : nullptr;
    ctx->in_slot = b;
  }
  const sagips_status s = sagips_train_step(ctx, step, flags, stream);
  if (ctx->in_noise || ctx->in_real) {  // slot b is free once the step's copies out of it are done
    ctx->in_noise = ctx->in_real = nullptr;
    CK(cudaEventRecord(ctx->in_free[ctx->in_slot], st));
    ctx->in_free_recorded[ctx->in_slot] = true;
  }
  if (s != SAGIPS_OK) return s;
  if (host_stats)
    CK(cudaMemcpyAsync(host_stats, ctx->stats, sizeof(sagips_step_stats), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  return SAGIPS_OK;
}

sagips_status sagips_push_generator_grad(sagips_ctx* ctx, uint64_t step, void* stream) {
  if (!ctx) return SAGIPS_ERR_INVALID_ARG;
  if (!ctx->have_step || ctx->local_done_step != step) return fail(ctx, SAGIPS_ERR_STATE, "push before train_step");
  sagips_status s = exchange_push(ctx, step, (cudaStream_t)stream);
  if (s != SAGIPS_OK) return s;
  ctx->pushed = true;
  return SAGIPS_OK;
}

sagips_status sagips_pull_generator_grad(sagips_ctx* ctx, uint64_t step, void* stream) {
  if (!ctx) return SAGIPS_ERR_INVALID_ARG;
  if (!ctx->pushed || ctx->local_done_step != step) return fail(ctx, SAGIPS_ERR_STATE, "pull before push");
  {
    const sagips_status xs = exchange_poll(ctx);
    if (xs != SAGIPS_OK) return xs;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (!ctx->skip_adam_once && exchange_fuses_adam(ctx, step)) {
    // wait + fold + Adam(G) in one kernel (the same arithmetic as below)
    const GenAdam ga = gen_adam_args(ctx);
    sagips_status s = exchange_pull(ctx, step, st, &ga);
    if (s != SAGIPS_OK) return s;
  } else {
    sagips_status s = exchange_pull(ctx, step, st);
    if (s != SAGIPS_OK) return s;
    if (ctx->skip_adam_once) {
      ctx->skip_adam_once = false;
    } else {
      adam_gen(ctx, st);
    }
  }
  mark(ctx, 7, st);
  if (timing_on(ctx)) ctx->timed_steps++;
  ctx->pushed = false;
  CK(cudaGetLastError());
  return SAGIPS_OK;
}

sagips_status sagips_phase_times(sagips_ctx* ctx, float* host_ms, int32_t n, int32_t* steps_averaged) {
  if (!ctx || !host_ms || n < SAGIPS_NUM_PHASES) return SAGIPS_ERR_INVALID_ARG;
  if (!ctx->cfg.phase_timing || ctx->timed_steps == 0) return fail(ctx, SAGIPS_ERR_STATE, "no timed steps");
  CK(cudaDeviceSynchronize());
  const int cnt = (int)std::min<int64_t>(ctx->timed_steps, sagips_ctx::kTimingRing);
  double acc[SAGIPS_NUM_PHASES] = {};
  for (int s = 0; s < cnt; ++s)
    for (int p = 0; p < SAGIPS_NUM_PHASES; ++p) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ctx->pev[s][p], ctx->pev[s][p + 1]));
      acc[p] += ms;
    }
  for (int p = 0; p < SAGIPS_NUM_PHASES; ++p) host_ms[p] = (float)(acc[p] / cnt);
  if (steps_averaged) *steps_averaged = cnt;
  return SAGIPS_OK;
}

sagips_status sagips_timing_reset(sagips_ctx* ctx) {
  if (!ctx) return SAGIPS_ERR_INVALID_ARG;
  CK(cudaDeviceSynchronize());
  ctx->timed_steps = 0;
  return SAGIPS_OK;
}

sagips_status sagips_kernel_times(sagips_ctx* ctx, float* host_ms, int32_t n, int32_t* steps_averaged) {
  if (!ctx || !host_ms || n < SAGIPS_NUM_KERNELS) return SAGIPS_ERR_INVALID_ARG;
  if (!ctx->cfg.phase_timing || ctx->timed_steps == 0) return fail(ctx, SAGIPS_ERR_STATE, "no timed steps");
  CK(cudaDeviceSynchronize());
  const int cnt = (int)std::min<int64_t>(ctx->timed_steps, sagips_ctx::kTimingRing);
  double acc[SAGIPS_NUM_KERNELS] = {};
  for (int s = 0; s < cnt; ++s)
    for (int i = 0; i < ctx->kcount[s]; ++i) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ctx->kev[s][i][0], ctx->kev[s][i][1]));
      const int k = ctx->kclass[s][i];
      if (k >= 0 && k < SAGIPS_NUM_KERNELS) acc[k] += ms;
    }
  for (int k = 0; k < SAGIPS_NUM_KERNELS; ++k) host_ms[k] = (float)(acc[k] / cnt);
  if (steps_averaged) *steps_averaged = cnt;
  return SAGIPS_OK;
}

static bool tensor_ref(sagips_ctx* c, int32_t which, void** p, size_t* bytes) {
  const auto& g = c->cfg;
  const int64_t k = g.param_samples, N = c->N;
  const int64_t hb = 4 * (g.hist_bins + 2);
  switch (which) {
    case SAGIPS_T_GEN_W: *p = c->gW; *bytes = 4 * c->G.nw; return true;
    case SAGIPS_T_GEN_B: *p = c->gB; *bytes = 4 * c->G.nb; return true;
    case SAGIPS_T_DISC_W: *p = c->dW; *bytes = 4 * c->D.nw; return true;
    case SAGIPS_T_DISC_B: *p = c->dB; *bytes = 4 * c->D.nb; return true;
    case SAGIPS_T_GEN_ADAM: *p = nullptr; *bytes = 4 * 2 * (c->G.nw + c->G.nb); return true;
    case SAGIPS_T_DISC_ADAM: *p = nullptr; *bytes = 4 * 2 * (c->D.nw + c->D.nb); return true;
    case SAGIPS_T_NOISE: *p = c->noise; *bytes = 4 * k * g.noise_dim; return true;
    case SAGIPS_T_RAW: *p = c->gAct[c->G.L - 1]; *bytes = 4 * 6 * k; return true;
    case SAGIPS_T_C: *p = c->cbuf; *bytes = 4 * 6 * k; return true;
    case SAGIPS_T_EVENTS: *p = c->X; *bytes = 4 * 4 * N; return true;
    case SAGIPS_T_REAL_IDX: *p = c->real_idx; *bytes = 4 * N; return true;
    case SAGIPS_T_HIST: *p = c->hist; *bytes = 4 * hb; return true;
    case SAGIPS_T_LOGITS_D: *p = c->logits_d; *bytes = 4 * 2 * N; return true;
    case SAGIPS_T_LOGITS_G: *p = c->logits_g; *bytes = 4 * N; return true;
    case SAGIPS_T_DY: *p = c->dy; *bytes = 4 * 2 * N; return true;
    case SAGIPS_T_DRAW: *p = c->draw; *bytes = 4 * 6 * k; return true;
    case SAGIPS_T_GEN_DW: *p = c->g_dW; *bytes = 4 * c->G.nw; return true;
    case SAGIPS_T_GEN_DB: *p = c->g_dB; *bytes = 4 * c->G.nb; return true;
    case SAGIPS_T_DISC_DW: *p = c->d_dW; *bytes = 4 * c->D.nw; return true;
    case SAGIPS_T_DISC_DB: *p = c->d_dB; *bytes = 4 * c->D.nb; return true;
    case SAGIPS_T_REDUCED: *p = c->reduced; *bytes = 4 * (c->G.nw + (c->cfg.packet_biases ? c->G.nb : 0)); return true;
    case SAGIPS_T_STATS: *p = c->stats; *bytes = sizeof(sagips_step_stats); return true;
    case SAGIPS_T_REFERENCE: *p = c->ref; *bytes = 4 * 2 * g.reference_rows; return true;
    case SAGIPS_T_SHARD: *p = c->shard; *bytes = 4 * 2 * g.shard_rows; return true;
    default: return false;
  }
}

sagips_status sagips_tensor_bytes(const sagips_ctx* ctx, int32_t which, size_t* bytes) {
  if (!ctx || !bytes) return SAGIPS_ERR_INVALID_ARG;
  void* p;
  return tensor_ref(const_cast<sagips_ctx*>(ctx), which, &p, bytes) ? SAGIPS_OK : SAGIPS_ERR_INVALID_ARG;
}

static sagips_status copy_adam(sagips_ctx* ctx, bool gen, void* host, bool to_host) {
  const MlpLayout& L = gen ? ctx->G : ctx->D;
  float* segs[4] = {gen ? ctx->gmW : ctx->dmW, gen ? ctx->gvW : ctx->dvW, gen ? ctx->gmB : ctx->dmB,
                    gen ? ctx->gvB : ctx->dvB};
  int64_t n[4] = {L.nw, L.nw, L.nb, L.nb};
  char* h = (char*)host;
  for (int i = 0; i < 4; ++i) {
    CK(to_host ? cudaMemcpy(h, segs[i], 4 * n[i], cudaMemcpyDeviceToHost)
               : cudaMemcpy(segs[i], h, 4 * n[i], cudaMemcpyHostToDevice));
    h += 4 * n[i];
  }
  return SAGIPS_OK;
}

sagips_status sagips_get(sagips_ctx* ctx, int32_t which, void* host, size_t bytes) {
  if (!ctx || !host) return SAGIPS_ERR_INVALID_ARG;
  void* p;
  size_t nb;
  if (!tensor_ref(ctx, which, &p, &nb) || nb != bytes)
    return fail(ctx, SAGIPS_ERR_INVALID_ARG, "tensor %d: size %zu != %zu", which, bytes, nb);
  CK(cudaDeviceSynchronize());
  if (which == SAGIPS_T_GEN_ADAM || which == SAGIPS_T_DISC_ADAM) return copy_adam(ctx, which == SAGIPS_T_GEN_ADAM, host, true);
  CK(cudaMemcpy(host, p, bytes, cudaMemcpyDeviceToHost));
  if (which == SAGIPS_T_STATS) {
    auto* s = reinterpret_cast<sagips_step_stats*>(host);
    s->step = ctx->last_step;
    if (s->nonfinite) return fail(ctx, SAGIPS_ERR_NONFINITE, "non-finite loss");
  }
  return exchange_check(ctx);
}

sagips_status sagips_set(sagips_ctx* ctx, int32_t which, const void* host, size_t bytes) {
  if (!ctx || !host) return SAGIPS_ERR_INVALID_ARG;
  void* p;
  size_t nb;
  if (!tensor_ref(ctx, which, &p, &nb) || nb != bytes)
    return fail(ctx, SAGIPS_ERR_INVALID_ARG, "tensor %d: size %zu != %zu", which, bytes, nb);
  CK(cudaDeviceSynchronize());
  if (which == SAGIPS_T_GEN_ADAM || which == SAGIPS_T_DISC_ADAM)
    return copy_adam(ctx, which == SAGIPS_T_GEN_ADAM, const_cast<void*>(host), false);
  CK(cudaMemcpy(p, host, bytes, cudaMemcpyHostToDevice));
  return SAGIPS_OK;
}

sagips_status sagips_debug_trace(void* host, size_t* bytes) {
  if (!bytes) return SAGIPS_ERR_INVALID_ARG;
  const size_t need = tc_trace_bytes();
  if (!host) {
    *bytes = need;
    return SAGIPS_OK;
  }
  if (*bytes != need) return SAGIPS_ERR_INVALID_ARG;
  if (cudaDeviceSynchronize() != cudaSuccess) return SAGIPS_ERR_CUDA;
  return tc_trace_copy(host) == 0 ? SAGIPS_OK : SAGIPS_ERR_CUDA;
}

sagips_status sagips_graph_stats(const sagips_ctx* ctx, uint64_t* graph_launches, uint64_t* instantiations) {
  if (!ctx || !graph_launches || !instantiations) return SAGIPS_ERR_INVALID_ARG;
  *graph_launches = ctx->graph_launches;
  *instantiations = ctx->graph_instantiations;
  return SAGIPS_OK;
}

sagips_status sagips_launch_count(const sagips_ctx* ctx, uint64_t* count) {
  if (!count) return SAGIPS_ERR_INVALID_ARG;
  *count = launches_total() - (ctx ? ctx->launch_base : 0);
  return SAGIPS_OK;
}

}  // extern "C"
