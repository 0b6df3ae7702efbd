// internal.h -- kernel launchers shared by the translation units of
// libsagips.so.  Not part of the public ABI (include/sagips.h is).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "common.cuh"

namespace sagips {

constexpr int kMaxLayers = 16;
constexpr int kMaxWorld = 64;
constexpr int kMaxSms = 256;  // bound on the persistent grids (B200: 148)

void count_launch();
uint64_t launches_total();

// k_tabulated.cu: the tabulated-CDF sampler variant (R32)
bool tabulated_ok(int G);
// hist (optional): [2 obs][bins+2] uint32 counts of the events (R22 bins), added atomically
void launch_sample_tabulated(const float* raw, int k, int m, int G, uint64_t seed, uint32_t step, uint32_t rank,
                             uint32_t stream_id, float* events, cudaStream_t st, uint32_t* hist = nullptr,
                             int bins = 0, const float* lo = nullptr, const float* hi = nullptr);
void launch_sample_tabulated_bwd(const float* raw, int k, int m, int G, uint64_t seed, uint32_t step, uint32_t rank,
                                 uint32_t stream_id, const float* dy, float* draw, cudaStream_t st);

// k_ensemble.cu: Eq. 6-8 over preds [M][k][P] -> out_dev [3][P] (p_hat, sigma, r_hat)
constexpr int kEnsMaxParams = 16;
int launch_ensemble_stats(const float* preds, int M, int k, int P, const double* p_true, double* out_dev,
                          cudaStream_t st);

struct Coef6 { float v[6]; };

// One Adam element (PyTorch form, R7): every Adam kernel uses this, so the
// fused exchange-fold + Adam(G) of exchange.cu is bitwise the same update.
__device__ __forceinline__ void adam_elem(float& p, float gi, float& m, float& v, float step_size, float bc2_sqrt,
                                          float b1, float b2, float eps) {
  const float mi = b1 * m + (1.f - b1) * gi;
  const float vi = b2 * v + (1.f - b2) * gi * gi;
  m = mi;
  v = vi;
  const float denom = sqrtf(vi) / bc2_sqrt + eps;
  p -= step_size * (mi / denom);
}

// Adam(G) operands of one step (sagips.cu gen_adam_args; advances tau)
struct GenAdam {
  float *pw, *mw, *vw;    // weights [nw]
  float *pb, *mb, *vb;    // biases [nb]
  const float* gb_local;  // local bias gradients (weights-only packet), else nullptr: biases are in the packet
  int64_t nw, nb;
  float step_size, bc2_sqrt, b1, b2, eps;
};

enum EpiKind { EPI_STORE = 0, EPI_BIAS_ACT = 1, EPI_ACT_GRAD = 2 };
struct Epi {
  int kind;
  const float* bias;  // EPI_BIAS_ACT
  int lrelu;          // EPI_BIAS_ACT: apply LeakyReLU
  float alpha;        // LeakyReLU slope
  const float* H;     // EPI_ACT_GRAD: post-activation whose sign selects 1 or alpha
  int ldh;
};

struct PacketList {
  const float* p[kMaxWorld];
  int count;
};

// k_data.cu
void launch_normals(float* out, int64_t count, float scale, uint64_t seed, uint32_t step, uint32_t rank,
                    uint32_t stream_id, cudaStream_t st);
void launch_reference(float* ref, int64_t n, const float c_true[6], uint64_t seed, cudaStream_t st);
void launch_shard(const float* ref, int64_t n_ref, float* shard, int64_t n_s, uint64_t seed, uint32_t rank,
                  cudaStream_t st);
void launch_constrain(const float* raw, float* c, int k, cudaStream_t st, bool tab = false);
void launch_sample_step(const float* c, int k, int m, const float* shard, int64_t n_shard, uint64_t seed,
                        uint32_t step, uint32_t rank, float* x_events, uint32_t* real_idx, uint32_t* hist,
                        int bins, const float lo[2], const float hi[2], cudaStream_t st, bool fake = true,
                        bool hist_zeroed = false);
void launch_sample_events(const float* c, int k, int m, uint64_t seed, uint32_t step, uint32_t rank,
                          uint32_t stream_id, float* events, uint32_t* hist, int bins, const float lo[2],
                          const float hi[2], cudaStream_t st);
// loss_part != nullptr: one extra block finishes a loss (finish_loss_block) instead of a k_finish_loss launch
struct LossFinish {
  const double* loss_part = nullptr;
  int nparts = 0;
  double scale = 0.0;
  float* out = nullptr;
  uint32_t* nonfinite = nullptr;
};
void launch_sample_bwd(const float* dy, const float* raw, int k, int m, uint64_t seed, uint32_t step,
                       uint32_t rank, float* draw, cudaStream_t st, const LossFinish& loss = LossFinish{});

// k_mlp_simt.cu
void launch_gemm(bool ta, bool tb, int M, int N, int K, const float* A, int lda, const float* B, int ldb,
                 float* C, int ldc, const Epi& ep, int splits, int64_t c_split, cudaStream_t st);
void launch_colsum(const float* X, int rows, int cols, int ldx, int splits, float* part, cudaStream_t st);
void launch_reduce_parts(const float* part, int nparts, int64_t n, float* out, float scale, cudaStream_t st);
int head_blocks();
void launch_head(const float* H, int M, int hd, const float* w, const float* b, int n_real, float label_rest,
                 float scale, float alpha, float* logits, float* dZprev, float* part, double* loss_part,
                 bool want_wgrad, cudaStream_t st);
void launch_finish_loss(const double* loss_part, int nparts, double scale, float* out, uint32_t* nonfinite,
                        cudaStream_t st);

// k_tc_gemm.cu (tcgen05, 128 -> 128 layers)
void launch_tc_rows(bool split, bool dgrad, const float* A, const float* W, float* C, int64_t rows, int epi,
                    const float* bias, const float* Hprev, float alpha, cudaStream_t st);
int tc_wgrad_grid();
void launch_tc_wgrad(bool split, const float* dZ, const float* H, int64_t rows, float* part, float* part_db,
                     cudaStream_t st);

// k_tc_layers.cu: warp-specialised tcgen05 layer passes on bf16 plane tiles
// (disc_depth >= 3; see the file header for the tensor formats), as one
// kernel per layer pass or as one pipelined kernel for the whole D / G step.
//
// A tensor of plane tiles: the whole tensor (slots == 0: tile t at t*TB) or a
// ring of `slots` tiles (tile t in slot t % slots) with per-tile counters:
// rdy[t] counts producer epilogue warps whose stores of tile t are complete
// (ready at 8), done[t] counts consumer completions (the slot may be
// overwritten by tile t + slots once done[t] == done_target).
struct Ring {
  uint8_t* base = nullptr;
  uint4* mask = nullptr;      // sign masks (hidden activations), [slots or tiles][128]
  uint32_t slots = 0;
  uint32_t* rdy = nullptr;
  uint32_t* done = nullptr;
  uint32_t done_target = 0;
};
struct FwdLaunch {
  Ring in;                     // input plane tiles (mid, head)
  Ring out;                    // output plane tiles (H + mask; head: G)
  Ring h1;                     // first, pipelined D step: H_1 planes for the backward (base == nullptr: none)
  uint32_t* tile_ctr = nullptr;  // middle layers: dynamic tile schedule counter (zeroed before the launch)
  const float* X = nullptr;    // [rows][2] (first)
  const float* W0 = nullptr;   // [128][2] (first)
  const float* b0 = nullptr;   // [128] (first)
  int first_help = 0;          // first: the epilogue warps produce H_1 rows 64-127 (else the producer warps do all)
  const float* W = nullptr;    // [128][128]
  const float* bias = nullptr;
  int64_t rows = 0;
  float alpha = 0.01f;
  const float* w_head = nullptr;
  const float* b_head = nullptr;
  int64_t n_real = 0;
  float label_rest = 0.f;
  float scale = 1.f;
  float* logits = nullptr;
  float* part_head = nullptr;  // [ctas][129]
  double* loss_part = nullptr; // [ctas]
  int want_wgrad = 0;
};
struct BwdLaunch {
  Ring g;                      // G_{l+1} plane tiles
  Ring h;                      // H_l plane tiles (wgrad, not first) + masks (not first)
  Ring gout;                   // G_l plane tiles (not first)
  const float* X = nullptr;
  const float* W0 = nullptr;
  const float* b0 = nullptr;
  const float* W = nullptr;
  int64_t rows = 0;
  float alpha = 0.01f;
  float* dy = nullptr;         // (first, no wgrad)
  float* part = nullptr;       // [ctas][128][128]
  float* part_db = nullptr;    // [ctas][128]
  float* part_l0 = nullptr;    // [ctas][384]
  uint32_t* tile_ctr = nullptr;  // no wgrad (G step): dynamic tile schedule counter (zeroed before the launch)
  // the fused D step's layer after the head (split): G = dz (Z > 0 ? w : alpha w)
  // generated in shared memory instead of loading g (k_tc_layers.cu kGenG)
  const float* gen_dz = nullptr;   // [rows_t] dz per row
  const uint4* gen_mask = nullptr; // [rows_t] sign bits of Z_4 (per-layer mask layout)
  const float* gen_w = nullptr;    // [128] head weights
};
enum { FWD_FIRST = 0, FWD_MID = 1, FWD_HEAD = 2 };
// k_fused.cu: the fused discriminator kernels (paper widths, depth 4)
struct GStepArgs {
  const float2* Y;         // [rows] fake events (D input rows)
  int64_t rows;
  const float* W[4];       // W_0 [128][2], W_1..W_3 [128][128]
  const float* b[4];       // b_0..b_3 [128]
  const float* w4;         // head [128]
  const float* b4;         // head bias [1]
  float alpha;
  float scale;             // 1 / N
  float* logits;           // [rows]
  double* loss_part;       // [grid]
  float2* dy;              // [rows]
  unsigned long long* trace;  // diagnostic (SAGIPS_FUSED_TRACE=1): CTA 0 phase stamps, else nullptr
};
struct DFwdArgs {
  const float2* X;         // [rows] D input rows (real then fake)
  int64_t rows;
  int64_t n_real;          // rows < n_real have label 1, the rest label_rest
  float label_rest;
  float scale;             // 1 / rows
  const float* W[4];       // W_0 [128][2], W_1..W_3 [128][128]
  const float* b[4];
  const float* w4;
  const float* b4;
  float alpha;
  float* logits;           // [rows]
  double* loss_part;       // [grid]
  float* part_head;        // [grid][129]: dW_head, db_head partials
  uint8_t* h2;             // H_2 plane tiles (hi plane written) + masks
  uint4* m2;
  uint8_t* h3;             // H_3 plane tiles (hi plane written) + masks
  uint4* m3;
  uint8_t* g4;             // G_4 plane tiles (hi + lo), or nullptr: dz and m4 instead (split)
  float* dz;               // [rows_t] dz per row (rows past the end: 0)
  uint4* m4;               // [rows_t] sign bits of Z_4 (per-layer mask layout)
  unsigned long long* trace;  // diagnostic (SAGIPS_FUSED_TRACE=1), else nullptr
};
int fused_grid(int64_t rows);
void launch_gstep(bool split, const GStepArgs& a, cudaStream_t st);
void launch_dfwd(bool split, const DFwdArgs& a, cudaStream_t st);
unsigned long long* fused_trace_buffer();  // nullptr unless SAGIPS_FUSED_TRACE=1
void fused_trace_report();                 // prints the phase breakdown of the last traced launch
int tc_layers_grid(int64_t rows);
size_t plane_tile_bytes(bool split);
void launch_tc_fwd(bool split, int kind, const FwdLaunch& L, cudaStream_t st);
void launch_tc_bwd(bool split, bool first, bool wgrad, const BwdLaunch& L, cudaStream_t st);
void launch_sum_parts(const float* part, int nparts, int64_t ld, int n, float* out, cudaStream_t st);
size_t tc_trace_bytes();
int tc_trace_copy(void* host);


// k_adam.cu
struct RedSeg {              // one parameter tensor: partials [nparts][ld] -> gradient g[n] -> Adam on p, m, v
  const float* part = nullptr;
  int64_t ld = 0;
  int nparts = 0;
  int n = 0;
  float *g = nullptr, *p = nullptr, *m = nullptr, *v = nullptr;
  int block0 = 0;            // (set by the launcher)
};
constexpr int kMaxRedSegs = 2 * kMaxLayers;
struct RedAdamArgs {
  RedSeg seg[kMaxRedSegs];
  int nseg = 0;
  // the D loss, finished by one extra block (instead of a k_finish_loss launch), or nullptr
  const double* loss_part = nullptr;
  int loss_nparts = 0;
  double loss_scale = 0.0;
  float* loss_out = nullptr;
  uint32_t* nonfinite = nullptr;
  int adam = 1;
  float step_size = 0.f, bc2_sqrt = 1.f, b1 = 0.f, b2 = 0.f, eps = 0.f;  // (set by the launcher)
};
void launch_reduce_adam(RedAdamArgs& a, double lr, int64_t tau, double b1, double b2, double eps, cudaStream_t st);
void launch_adam(float* p, const float* g, float* m, float* v, int64_t n, double lr, int64_t tau, double b1,
                 double b2, double eps, cudaStream_t st);
void launch_fold(const PacketList& pl, int64_t n, float* out, float divisor, cudaStream_t st);

}  // namespace sagips
