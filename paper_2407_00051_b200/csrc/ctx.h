// ctx.h -- the rank context (host struct) behind the opaque sagips_ctx.
#pragma once
#include <cuda_runtime.h>

#include <string>

#include "../../include/sagips.h"
#include "internal.h"

namespace sagips {

struct MlpLayout {
  int L = 0;                    // linear layers
  int sizes[kMaxLayers + 1] = {};
  int64_t w_off[kMaxLayers] = {}, b_off[kMaxLayers] = {};
  int64_t nw = 0, nb = 0;       // weights / biases
  int maxw = 0;                 // widest layer
  void build(int in, int hidden, int depth, int out);
};

struct ExchangeState;  // exchange.cu
struct TcState;        // k_disc_tc.cu

}  // namespace sagips

struct sagips_ctx {
  sagips_config cfg{};
  int dev = 0;
  std::string err;
  sagips::MlpLayout G, D;
  int64_t N = 0;
  size_t ws_bytes = 0;
  uint64_t launch_base = 0;
  // parameters and Adam state (fp32 masters)
  float *gW = nullptr, *gB = nullptr, *gmW = nullptr, *gvW = nullptr, *gmB = nullptr, *gvB = nullptr;
  float *dW = nullptr, *dB = nullptr, *dmW = nullptr, *dvW = nullptr, *dmB = nullptr, *dvB = nullptr;
  // gradients; g_dW is the weights-only packet
  float *g_dW = nullptr, *g_dB = nullptr, *d_dW = nullptr, *d_dB = nullptr, *reduced = nullptr;
  // data
  float *ref = nullptr, *shard = nullptr;
  // generator activations
  float* noise = nullptr;
  float* gAct[sagips::kMaxLayers] = {};
  float* gdZ[2] = {};
  float* gdz_all[sagips::kMaxLayers] = {};  // fused generator backward: dZ of every hidden layer
  float *cbuf = nullptr, *draw = nullptr;
  // discriminator input/activations (fp32 path)
  float* X = nullptr;
  uint32_t* real_idx = nullptr;
  float* dAct[sagips::kMaxLayers] = {};
  uint4* dMask[sagips::kMaxLayers] = {};  // sign masks of the hidden activations (tcgen05 layers)
  float* dZb[2] = {};
  float *logits_d = nullptr, *logits_g = nullptr, *dy = nullptr;
  uint32_t* hist = nullptr;
  float* part = nullptr;
  int64_t part_floats = 0;
  float* colpart = nullptr;
  float* head_tmp = nullptr;
  float* dbpart = nullptr;  // [grid][128] bias-gradient partials (tcgen05 layers)
  float* lpart[sagips::kMaxLayers] = {};  // [ctas][128][128] wgrad partials of hidden layer l
  float* ldb[sagips::kMaxLayers] = {};    // [ctas][128] bias-gradient partials
  bool d_adam_done = false;               // the D step already applied Adam(D) (fused reduction)
  // sagips_train_step_host: the caller's inputs are copied on copy_stream
  // into staging buffer b = step & 1 (so the copy of step t+1 overlaps step
  // t), the step copies them into place on its own stream
  const float* in_noise = nullptr;        // this step's staged inputs (device), or nullptr
  const float* in_real = nullptr;
  float* hin[2] = {};                     // [k d noise | 2 N real] per slot
  int in_slot = 0;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t in_ready[2] = {}, in_free[2] = {};
  bool in_free_recorded[2] = {};
  static constexpr int kTileCtrs = 16;
  uint32_t* tile_ctrs = nullptr;          // dynamic tile-schedule counters of the layer kernels
  int tile_ctr_next = 0;
  double* loss_part = nullptr;
  int loss_g_defer = 0;                   // fused G step: L_G's partials, finished by the sampler backward's extra block
  double loss_g_scale = 0.0;
  sagips_step_stats* stats = nullptr;
  // step bookkeeping
  int64_t g_tau = 0, d_tau = 0;
  bool use_tc = false;  // discriminator 128 -> 128 layers on tcgen05
  bool have_step = false;
  uint64_t last_step = 0;
  uint64_t local_done_step = ~0ull;
  bool pushed = false;
  bool skip_adam_once = false;
  sagips::ExchangeState* xs = nullptr;
  // CUDA-graph step (SAGIPS_STEP_GRAPH): the step is captured and replayed;
  // phase / kernel timing events are not recorded while capturing
  bool capturing = false;
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cstream = nullptr;  // capture stream
  uint64_t graph_launches = 0, graph_instantiations = 0;
  sagips::TcState* tc = nullptr;
  // phase timing: events at the SAGIPS_NUM_PHASES+1 boundaries of the
  // last 64 steps (cfg.phase_timing)
  static constexpr int kTimingRing = 64;
  cudaEvent_t pev[kTimingRing][SAGIPS_NUM_PHASES + 1] = {};
  int64_t timed_steps = 0;
  int pslot = 0;
  // per-kernel timing of the tensor-core layer passes (sagips_kernel_times):
  // start/stop events per launch, up to kKernelSlots launches per step
  static constexpr int kKernelSlots = 16;
  cudaEvent_t kev[kTimingRing][kKernelSlots][2] = {};
  int kclass[kTimingRing][kKernelSlots] = {};
  int kcount[kTimingRing] = {};
};

namespace sagips {
inline bool timing_on(const sagips_ctx* c) { return c->cfg.phase_timing && !c->capturing; }
inline void mark(sagips_ctx* c, int boundary, cudaStream_t st) {
  if (timing_on(c)) cudaEventRecord(c->pev[c->pslot][boundary], st);
}
// bracket one kernel launch of class k (SAGIPS_NUM_KERNELS) with events
inline void kernel_begin(sagips_ctx* c, int k, cudaStream_t st) {
  if (!timing_on(c)) return;
  const int i = c->kcount[c->pslot];
  if (i >= sagips_ctx::kKernelSlots) return;
  if (!c->kev[c->pslot][i][0]) {
    cudaEventCreate(&c->kev[c->pslot][i][0]);
    cudaEventCreate(&c->kev[c->pslot][i][1]);
  }
  c->kclass[c->pslot][i] = k;
  cudaEventRecord(c->kev[c->pslot][i][0], st);
}
inline void kernel_end(sagips_ctx* c, cudaStream_t st) {
  if (!timing_on(c)) return;
  const int i = c->kcount[c->pslot];
  if (i >= sagips_ctx::kKernelSlots) return;
  cudaEventRecord(c->kev[c->pslot][i][1], st);
  c->kcount[c->pslot] = i + 1;
}
}  // namespace sagips

namespace sagips {
void adam_gen(sagips_ctx* c, cudaStream_t st);
// k_gen.cu: fused generator passes (widths <= 128)
bool gen_fused_ok(const sagips_ctx* c);
// noise_step != nullptr: a1 too -- the forward draws the step's noise into c->noise itself
void launch_gen_fwd(sagips_ctx* c, cudaStream_t st, const void* prefetch = nullptr, int64_t prefetch_bytes = 0,
                    uint32_t* zero_hist = nullptr, int zero_words = 0, const uint32_t* noise_step = nullptr);
// the generator forward on a caller-given noise batch (k <= param_samples rows):
// the constrained parameters -> c_out [k][6]; reuses the step's activation buffers
void launch_gen_predict(sagips_ctx* c, const float* noise, int k, float* c_out, cudaStream_t st);
void launch_gen_bwd(sagips_ctx* c, cudaStream_t st);
// exchange.cu
sagips_status exchange_push(sagips_ctx* c, uint64_t step, cudaStream_t st);
// adam (optional): when exchange_fuses_adam(c, step), pull runs the wait,
// the fold and Adam(G) in one kernel with these operands
sagips_status exchange_pull(sagips_ctx* c, uint64_t step, cudaStream_t st, const GenAdam* adam = nullptr);
bool exchange_fuses_adam(const sagips_ctx* c, uint64_t step);
GenAdam gen_adam_args(sagips_ctx* c);
sagips_status exchange_check(sagips_ctx* c);
sagips_status exchange_poll(sagips_ctx* c);
// graph capture support: whether this configuration's step can be captured,
// and the join of the exchange side stream into the step stream
bool exchange_graph_ok(const sagips_ctx* c);
bool exchange_outer_step(const sagips_ctx* c, uint64_t step);
sagips_status exchange_join(sagips_ctx* c, cudaStream_t st);  // non-blocking: an error raised by an earlier wait
void exchange_destroy(sagips_ctx* c);
}  // namespace sagips
