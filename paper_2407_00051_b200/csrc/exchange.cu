// exchange.cu -- the asynchronous ring exchange of generator weight
// gradients between GPUs, B200-native:
//
//  * one-sided ring (RMA-ARAR): every rank owns a window of
//    version-indexed packet slots in its HBM, cudaMalloc'ed here and mapped
//    into every peer over NVLink/NVSwitch by CUDA IPC.  push(t) stores the
//    packet straight into the successor's slot and publishes it with a
//    release store of the tag t+1 (the writer never waits); a
//    forwarding agent on a high-priority side stream passes the packets of
//    the other origins along the ring as they land (Alg. 1, R10);
//    pull(t) waits (bounded, acquire loads) for the packets it needs and
//    folds them in ascending origin order.
//  * two-sided ring (ARAR): the same pass-along schedule with
//    ncclSend/ncclRecv on the side stream.
//  * outer leaders' ring every h steps (R13): NCCL send/recv
//    among the first rank of each inner group.
//  * one-hop all-gather (SAGIPS_MODE_RMA_ALLGATHER, §8(f) row 3): push(t)
//    stores the packet into every group member's window at once (NVSwitch
//    gives every pair a direct path); pull is the same wait + ascending fold.
//  * SYNC_ALLREDUCE: ncclAllReduce (the synchronous baseline).
//  * staleness s (R12): pull(t) folds the own packet of step t with the
//    others' packets of step t-s, so with s = 1 the ring of step t runs on
//    the side stream while step t+1 computes.
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <vector>

#include <nccl.h>

#include "ctx.h"

namespace sagips {

constexpr int kVersions = 4;  // slot depth: >= 2 + 2s (exchange)
enum { RING_INNER = 0 };

struct DevFlags {
  unsigned long long tag[kMaxWorld][kVersions];
  unsigned long long tag_ag[kMaxWorld][kVersions];  // RMA_CHUNKED: the reduced chunk of member q landed
};

struct ExchangeState {
  int pos = 0, g = 1;            // position in the inner group, its size (the last group may be smaller)
  int first = 0;                 // first rank of the inner group
  int nlead = 1;                 // inner groups = leaders = ceil(world / group_size)
  int succ = 0, pred = 0;        // ring neighbours (global ranks)
  // one-sided window: slots[origin][version][Pw] fp32 + flags
  float* win = nullptr;          // own window (cudaMalloc, IPC-exported)
  DevFlags* flags = nullptr;     // own flags (inside the same allocation)
  size_t win_bytes = 0;
  cudaIpcMemHandle_t handle{};
  bool have_handle = false;
  char* peer_base[kMaxWorld] = {};
  bool peers_ok = false;
  bool local_peers = false;      // sagips_connect_peers_local: raw pointers of one process (no IPC)
  // two-sided / outer / sync
  ncclComm_t comm_ring = nullptr;   // side-stream ring
  ncclComm_t comm_main = nullptr;   // outer ring and all-reduce (main stream)
  float* gather[2] = {nullptr, nullptr};  // [g][Pw] per version parity
  float* outer_buf = nullptr;              // [n_leaders][Pw]
  // streams/events
  cudaStream_t side = nullptr;
  cudaEvent_t ev_ready[2] = {nullptr, nullptr};
  cudaEvent_t ev_done[2] = {nullptr, nullptr};
  bool ring_issued[2] = {false, false};
  uint64_t ring_step[2] = {0, 0};
  // device error word and wait accounting
  unsigned int* err = nullptr;      // device: 1 timeout, 2 protocol
  unsigned int* herr = nullptr;     // the same code in mapped pinned host memory (read without a sync)
  unsigned int* herr_dev = nullptr; // its device alias
  unsigned int* ticket = nullptr;   // device [kMaxWorld]: k_push's last-CTA counters (self-resetting)
  uint32_t* one = nullptr;          // device constant 1 (stats.outer_fired)
};

// the packet: generator weight gradients, plus the bias gradients with the fused packet
static size_t slot_floats(const sagips_ctx* c) { return (size_t)c->G.nw + (c->cfg.packet_biases ? c->G.nb : 0); }
// distance between packets in windows and buffers: 256-byte aligned (float4
// copies; the fused packet's length is not a multiple of 4)
static size_t slot_stride(const sagips_ctx* c) { return (slot_floats(c) + 63) & ~(size_t)63; }

static float* slot_ptr(char* base, const sagips_ctx* c, int origin, uint64_t version) {
  const size_t per_origin = kVersions * slot_stride(c);
  return reinterpret_cast<float*>(base) + origin * per_origin + (version % kVersions) * slot_stride(c);
}
static DevFlags* flags_ptr(char* base, const sagips_ctx* c) {
  return reinterpret_cast<DevFlags*>(base + sizeof(float) * (size_t)c->cfg.world * kVersions * slot_stride(c));
}

// ---------------------------------------------------------------- device side
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Error codes: 1 timeout, 2 protocol (slot overrun).  The device word gates
// the fold/Adam kernel of the same step; the host-mapped copy lets the next
// API call report the error without synchronising.
struct ErrWords {
  unsigned int* dev;
  unsigned int* host;  // device alias of mapped pinned host memory
};
__device__ __forceinline__ void raise_err(ErrWords e, unsigned int code) {
  atomicExch(e.dev, code);
  *reinterpret_cast<volatile unsigned int*>(e.host) = code;
  __threadfence_system();
}

// Wait until *flag >= want; returns false on timeout (raises 1).
__device__ bool wait_tag(const unsigned long long* flag, unsigned long long want, unsigned long long timeout_ns,
                         ErrWords err) {
  const unsigned long long t0 = globaltimer();
  while (ld_acquire_sys(flag) < want) {
    if (globaltimer() - t0 > timeout_ns) {
      raise_err(err, 1u);
      return false;
    }
    __nanosleep(64);
  }
  return true;
}

// Block-wide copy of n floats (16-byte aligned).
__device__ void block_copy(float* __restrict__ dst, const float* __restrict__ src, int64_t n) {
  const int64_t n4 = n / 4;
  const float4* s4 = reinterpret_cast<const float4*>(src);
  float4* d4 = reinterpret_cast<float4*>(dst);
  for (int64_t i = threadIdx.x; i < n4; i += blockDim.x) d4[i] = s4[i];
  for (int64_t i = 4 * n4 + threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// push: the own packet -> destination y's slot (origin = me), then release
// its tag.  y = blockIdx.y: the successor (pass-along ring) or every other
// member (one-hop all-gather, SAGIPS_MODE_RMA_ALLGATHER: over NVSwitch every
// member is one hop away, so there is no forwarding agent).  push_ctas CTAs
// per destination each store one contiguous chunk (round 1, torch.profiler
// at N = 2: 14.7 us with one CTA, ~10 us with 8-148 CTAs -- a ~9 us floor
// that remains without the fences, so not the store bandwidth).
// The last CTA to finish (ticket counter, reset by it) publishes the tag:
// every CTA fences its stores before taking a ticket, the last fences again
// before the release store.
// CTAs per destination: at least 32 (the paper's 200 KB packet: 13 CTAs of
// one unrolled round each measured 15.4 vs 13.3 us), up to 4 x 148 for large
// packets, each thread moving 4 float4 per round trip
static int push_ctas(int64_t n_floats) {
  return (int)std::max<int64_t>(32, std::min<int64_t>((n_floats / 4 + 1023) / 1024, 4 * 148));
}
struct PushAllArgs {
  float* dst[kMaxWorld];
  unsigned long long* dst_flag[kMaxWorld];
  int64_t off[kMaxWorld];  // source offset and length per destination (RMA_CHUNKED: chunk y; else 0, n)
  int64_t len[kMaxWorld];
};
__global__ void __launch_bounds__(256) k_push(const float* __restrict__ packet_base, int64_t n_unused, PushAllArgs a,
                                              unsigned long long tag, unsigned int* ticket) {
  const int y = blockIdx.y;
  float* dst = a.dst[y];
  const float* packet = packet_base + a.off[y];
  const int64_t n = a.len[y];
  const int64_t n4 = n / 4, per = (n4 + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per, b1 = min(n4, b0 + per);
  const float4* s4 = reinterpret_cast<const float4*>(packet);
  float4* d4 = reinterpret_cast<float4*>(dst);
  // four independent loads in flight per thread before their remote stores
  for (int64_t i = b0 + threadIdx.x; i < b1; i += 4 * blockDim.x) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u * blockDim.x < b1) v[u] = s4[i + u * blockDim.x];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i + u * blockDim.x < b1) d4[i + u * blockDim.x] = v[u];
  }
  if (blockIdx.x == gridDim.x - 1)
    for (int64_t i = 4 * n4 + threadIdx.x; i < n; i += blockDim.x) dst[i] = packet[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(&ticket[y], 1u) == gridDim.x - 1) {
      ticket[y] = 0;
      __threadfence_system();
      st_release_sys(a.dst_flag[y], tag);
    }
  }
}

struct FwdArgs {
  float* src[kMaxWorld];               // own window slots, in hop order
  float* dst[kMaxWorld];               // successor's slots
  unsigned long long* src_flag[kMaxWorld];
  unsigned long long* dst_flag[kMaxWorld];
  int hops;
};

// forwarding agent: for hop j, wait for the packet of origin pos-j in the own
// window, then pass it to the successor (Alg. 1's "send to rank i+1").
// Register budget: at most 32 per thread (min 2 blocks/SM), so the agent's
// 1024 threads fit on an SM beside the spinning CTAs of k_wait_fold_adam.
// With 64 (the 1024-thread cap) it needed a whole SM's register file; at
// g >= 3, staleness 0 and C2 sizes the fused pull puts a CTA on every SM and
// waits for packets that the peers' starved agents never forward (measured:
// exchange wait timeout at N = 4).
__global__ void __launch_bounds__(1024, 2) k_forward(FwdArgs a, int64_t n, unsigned long long tag,
                                                  unsigned long long timeout_ns, ErrWords err) {
  __shared__ int ok;
  for (int j = 0; j < a.hops; ++j) {
    if (threadIdx.x == 0) ok = wait_tag(a.src_flag[j], tag, timeout_ns, err);
    __syncthreads();
    if (!ok) return;
    block_copy(a.dst[j], a.src[j], n);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      st_release_sys(a.dst_flag[j], tag);
    }
  }
}

struct WaitArgs {
  unsigned long long* flag[kMaxWorld];
  unsigned long long want[kMaxWorld];
  int count;
};

// The wait of a pull: ONE thread waits (bounded) for the tags it needs and
// checks that no newer packet overwrote a slot (protocol error 2).  Only this
// one-warp CTA spins, so the ring's forwarding agents (and any other work)
// always find room on the SMs while a rank waits for its peers.
__global__ void k_wait(WaitArgs a, unsigned long long timeout_ns, ErrWords err, unsigned long long* wait_ns,
                       uint32_t* outer_fired) {
  if (threadIdx.x != 0) return;
  const unsigned long long t0 = globaltimer();
  for (int i = 0; i < a.count; ++i) {
    if (!wait_tag(a.flag[i], a.want[i], timeout_ns, err)) break;
    if (ld_acquire_sys(a.flag[i]) != a.want[i]) raise_err(err, 2u);  // a newer packet overwrote the slot
  }
  if (wait_ns) *wait_ns = globaltimer() - t0;
  if (outer_fired) *outer_fired = 0u;
}

// The fold of a pull and (optionally) Adam(G), launched after k_wait with
// programmatic dependent launch (its launch overlaps the wait; griddepcontrol
// .wait orders it after k_wait's writes).  If a wait of this step failed
// (err != 0) nothing is written: the generator keeps its weights and the
// host reports the error at the next call (sagips_train_step / pull).
// Per element: the ascending fold reduced[i] = (sum_j p_j[i]) / divisor for
// i < pw (loads through L2: peers wrote the slots) and the Adam update of
// adam_elem, as k_adam -- weights from reduced[i], biases from reduced[nw+j]
// (fused packet) or the local gradient.
struct FoldAdamArgs {
  PacketList pl;
  float* reduced;
  int64_t pw;
  float divisor;
  int do_adam;
  GenAdam a;
  const unsigned int* err;
  int64_t gather_chunk;  // RMA_CHUNKED: element i is already reduced, in pl.p[i / gather_chunk][i]; 0: fold
  int vec;               // every array 16-byte aligned: the weights go four at a time (a multiple-of-64 chunk never splits a quad)
  uint32_t* zero_word;   // written 0 by one thread (the stats' outer-ring flag of a step without exchange), or nullptr
};
__device__ __forceinline__ float4 ldcg4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }
__global__ void __launch_bounds__(256) k_fold_adam(const __grid_constant__ FoldAdamArgs f) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (f.zero_word && blockIdx.x == 0 && threadIdx.x == 0) *f.zero_word = 0u;
  if (f.err && *reinterpret_cast<const volatile unsigned int*>(f.err) != 0u) return;
  const GenAdam& a = f.a;
  const int64_t n = f.do_adam ? a.nw + a.nb : f.pw;
  // large packets: quads (the same per-element arithmetic and fold order)
  const int64_t nq = f.vec ? (f.do_adam ? (f.pw < a.nw ? f.pw : a.nw) : f.pw) >> 2 : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += stride) {
    const int64_t i = 4 * q;
    float4 g;
    if (f.gather_chunk) {
      g = ldcg4(f.pl.p[i / f.gather_chunk] + i);
    } else {
      float4 acc = ldcg4(f.pl.p[0] + i);
      for (int j = 1; j < f.pl.count; ++j) {
        const float4 u = ldcg4(f.pl.p[j] + i);
        acc.x += u.x; acc.y += u.y; acc.z += u.z; acc.w += u.w;
      }
      g = make_float4(acc.x / f.divisor, acc.y / f.divisor, acc.z / f.divisor, acc.w / f.divisor);
    }
    *reinterpret_cast<float4*>(f.reduced + i) = g;
    if (!f.do_adam) continue;
    float4 p = *reinterpret_cast<const float4*>(a.pw + i), m = *reinterpret_cast<const float4*>(a.mw + i),
           v = *reinterpret_cast<const float4*>(a.vw + i);
    adam_elem(p.x, g.x, m.x, v.x, a.step_size, a.bc2_sqrt, a.b1, a.b2, a.eps);
    adam_elem(p.y, g.y, m.y, v.y, a.step_size, a.bc2_sqrt, a.b1, a.b2, a.eps);
    adam_elem(p.z, g.z, m.z, v.z, a.step_size, a.bc2_sqrt, a.b1, a.b2, a.eps);
    adam_elem(p.w, g.w, m.w, v.w, a.step_size, a.bc2_sqrt, a.b1, a.b2, a.eps);
    *reinterpret_cast<float4*>(a.pw + i) = p;
    *reinterpret_cast<float4*>(a.mw + i) = m;
    *reinterpret_cast<float4*>(a.vw + i) = v;
  }
  for (int64_t i = 4 * nq + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    float gi = 0.f;
    if (i < f.pw) {
      if (f.gather_chunk) {
        gi = __ldcg(f.pl.p[i / f.gather_chunk] + i);
      } else {
        float acc = __ldcg(f.pl.p[0] + i);
        for (int j = 1; j < f.pl.count; ++j) acc += __ldcg(f.pl.p[j] + i);
        gi = acc / f.divisor;
      }
      f.reduced[i] = gi;
    }
    if (!f.do_adam) continue;
    if (i < a.nw) {
      float p = a.pw[i], m = a.mw[i], v = a.vw[i];
      adam_elem(p, gi, m, v, a.step_size, a.bc2_sqrt, a.b1, a.b2, a.eps);
      a.pw[i] = p;
      a.mw[i] = m;
      a.vw[i] = v;
    } else {
      const int64_t j = i - a.nw;
      float p = a.pb[j], m = a.mb[j], v = a.vb[j];
      adam_elem(p, a.gb_local ? a.gb_local[j] : gi, m, v, a.step_size, a.bc2_sqrt, a.b1, a.b2, a.eps);
      a.pb[j] = p;
      a.mb[j] = m;
      a.vb[j] = v;
    }
  }
}

// RMA_CHUNKED reduce-scatter step of member q: chunk q of every member's
// packet, folded in ascending origin order (the same element-wise sum as
// k_fold_adam's fold), divided, and stored into every member's window (the
// all-gather); the last CTA releases the chunk's tag in the peers' windows.
// Launched after k_wait (programmatic dependent launch).
struct RsArgs {
  PacketList pl;                      // the group's packets in ascending origin order
  float* dst[kMaxWorld];              // the reduced chunk's destination in every member's window (own first)
  unsigned long long* flag[kMaxWorld];// its tag in the peers' windows (dst[d], d >= 1)
  int ndst;
  int64_t off, len;                   // the chunk
  float divisor;
  unsigned long long tag;
  unsigned int* ticket;
  const unsigned int* err;
  int vec;                            // every pointer 16-byte aligned
};
__global__ void __launch_bounds__(256) k_rs_fold(const __grid_constant__ RsArgs a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (*reinterpret_cast<const volatile unsigned int*>(a.err) != 0u) return;  // the peers' waits time out (bounded)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nq = a.vec ? a.len >> 2 : 0;  // quads (off is a multiple of 64 floats)
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nq; k += stride) {
    const int64_t i = a.off + 4 * k;
    float4 acc = ldcg4(a.pl.p[0] + i);
    for (int j = 1; j < a.pl.count; ++j) {
      const float4 u = ldcg4(a.pl.p[j] + i);
      acc.x += u.x; acc.y += u.y; acc.z += u.z; acc.w += u.w;
    }
    const float4 v = make_float4(acc.x / a.divisor, acc.y / a.divisor, acc.z / a.divisor, acc.w / a.divisor);
    for (int d = 0; d < a.ndst; ++d) *reinterpret_cast<float4*>(a.dst[d] + i) = v;
  }
  for (int64_t k = 4 * nq + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < a.len; k += stride) {
    const int64_t i = a.off + k;
    float acc = __ldcg(a.pl.p[0] + i);
    for (int j = 1; j < a.pl.count; ++j) acc += __ldcg(a.pl.p[j] + i);
    const float v = acc / a.divisor;
    for (int d = 0; d < a.ndst; ++d) a.dst[d][i] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(a.ticket, 1u) == gridDim.x - 1) {
      *a.ticket = 0;
      __threadfence_system();
      for (int d = 1; d < a.ndst; ++d) st_release_sys(a.flag[d], a.tag);
    }
  }
}

static cudaError_t launch_fold_adam(FoldAdamArgs f, cudaStream_t st) {
  auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  bool vec = a16(f.reduced);
  for (int j = 0; j < f.pl.count; ++j) vec = vec && a16(f.pl.p[j]);
  if (f.do_adam) vec = vec && a16(f.a.pw) && a16(f.a.mw) && a16(f.a.vw);
  const int64_t n = f.do_adam ? f.a.nw + f.a.nb : f.pw;
  // quads for large packets only: at the paper's 50 K parameters one element
  // per thread over more CTAs has the shorter critical path (latency-bound)
  f.vec = (vec && n >= (int64_t(1) << 20)) ? 1 : 0;
  const int64_t per_thread = f.vec ? 4 : 1;  // f.vec set above
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)std::min<int64_t>((n / per_thread + 255) / 256, 148 * 8));
  lc.blockDim = dim3(256);
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&lc, k_fold_adam, f);
  count_launch();
  return e;
}

// ---------------------------------------------------------------- host side
#define XCK(call)                                                                          \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      c->err = std::string(#call) + ": " + cudaGetErrorString(e_);                         \
      return SAGIPS_ERR_CUDA;                                                              \
    }                                                                                      \
  } while (0)
#define NCK(call)                                                                          \
  do {                                                                                     \
    ncclResult_t r_ = (call);                                                              \
    if (r_ != ncclSuccess) {                                                               \
      c->err = std::string(#call) + ": " + ncclGetErrorString(r_);                         \
      return SAGIPS_ERR_CUDA;                                                              \
    }                                                                                      \
  } while (0)

static bool one_sided(const sagips_ctx* c) {
  return c->cfg.mode == SAGIPS_MODE_RMA_ARAR_ARAR || c->cfg.mode == SAGIPS_MODE_RMA_ALLGATHER ||
         c->cfg.mode == SAGIPS_MODE_RMA_CHUNKED;
}
// RMA_CHUNKED: chunk q of the packet = [q cs, min(n, (q + 1) cs)), cs a multiple of 64 floats
static int64_t chunk_floats(const sagips_ctx* c, int g) {
  const int64_t n = (int64_t)slot_floats(c);
  return ((n + g - 1) / g + 63) / 64 * 64;
}
// the leaders' outer ring through the windows (one-hop all-gather, cfg.outer_rma)
static bool outer_one_sided(const sagips_ctx* c) { return one_sided(c) && c->cfg.outer_rma != 0; }
static int n_leaders(const sagips_config& g) { return (g.world + g.group_size - 1) / g.group_size; }
static bool is_leader(const sagips_config& g) { return g.rank % g.group_size == 0; }
static bool needs_nccl(const sagips_ctx* c) {
  const auto& g = c->cfg;
  if (g.world == 1 || g.mode == SAGIPS_MODE_NONE) return false;
  if (one_sided(c)) return !outer_one_sided(c) && g.outer_every > 0 && g.group_size < g.world;
  return true;
}
// ranks whose window this rank maps: its inner group, and the other leaders
// when it is a leader with the one-sided outer ring
static bool maps_peer(const sagips_ctx* c, int q) {
  const auto& g = c->cfg;
  const ExchangeState* x = c->xs;
  if (q >= x->first && q < x->first + x->g) return true;
  return outer_one_sided(c) && is_leader(g) && q % g.group_size == 0 && g.outer_every > 0;
}

static sagips_status ensure_state(sagips_ctx* c) {
  if (c->xs) return SAGIPS_OK;
  auto* x = new ExchangeState();
  c->xs = x;
  const auto& g = c->cfg;
  int gs = g.group_size;
  if (g.mode == SAGIPS_MODE_ARAR) gs = g.world;  // ungrouped
  x->first = (g.rank / gs) * gs;
  x->g = std::min(gs, g.world - x->first);  // contiguous groups; the last may be smaller
  x->pos = g.rank - x->first;
  x->succ = x->first + (x->pos + 1) % x->g;
  x->pred = x->first + (x->pos + x->g - 1) % x->g;
  x->nlead = n_leaders(g);
  int lo, hi;
  XCK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  XCK(cudaStreamCreateWithPriority(&x->side, cudaStreamNonBlocking, hi));
  for (int i = 0; i < 2; ++i) {
    XCK(cudaEventCreateWithFlags(&x->ev_ready[i], cudaEventDisableTiming));
    XCK(cudaEventCreateWithFlags(&x->ev_done[i], cudaEventDisableTiming));
  }
  XCK(cudaMalloc(&x->err, sizeof(unsigned int)));
  XCK(cudaMemset(x->err, 0, sizeof(unsigned int)));
  XCK(cudaHostAlloc(&x->herr, sizeof(unsigned int), cudaHostAllocMapped));
  *reinterpret_cast<volatile unsigned int*>(x->herr) = 0u;
  XCK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&x->herr_dev), x->herr, 0));
  XCK(cudaMalloc(&x->ticket, sizeof(unsigned int) * kMaxWorld));
  XCK(cudaMemset(x->ticket, 0, sizeof(unsigned int) * kMaxWorld));
  XCK(cudaMalloc(&x->one, sizeof(uint32_t)));
  const uint32_t one = 1;
  XCK(cudaMemcpy(x->one, &one, sizeof one, cudaMemcpyHostToDevice));
  if (g.world > 1 && g.mode != SAGIPS_MODE_NONE) {
    const size_t ps = slot_stride(c);
    XCK(cudaMalloc(&x->gather[0], sizeof(float) * ps * gs));
    XCK(cudaMalloc(&x->gather[1], sizeof(float) * ps * gs));
    XCK(cudaMalloc(&x->outer_buf, sizeof(float) * ps * std::max(x->nlead, 1)));
    if (one_sided(c)) {
      // slots[origin][version]: inner-group origins carry packets, other
      // leaders' origins carry their inner sums (one-sided outer ring)
      x->win_bytes = sizeof(float) * (size_t)g.world * kVersions * ps + sizeof(DevFlags);
      XCK(cudaMalloc(&x->win, x->win_bytes));
      XCK(cudaMemset(x->win, 0, x->win_bytes));
      x->flags = flags_ptr(reinterpret_cast<char*>(x->win), c);
      XCK(cudaIpcGetMemHandle(&x->handle, x->win));
      x->have_handle = true;
    }
  }
  return SAGIPS_OK;
}

static ErrWords err_words(const ExchangeState* x) { return ErrWords{x->err, x->herr_dev}; }

static sagips_status err_status(sagips_ctx* c, unsigned int e) {
  if (e == 1) { c->err = "exchange wait timed out"; return SAGIPS_ERR_TIMEOUT; }
  if (e == 2) { c->err = "exchange slot overrun (protocol)"; return SAGIPS_ERR_PROTOCOL; }
  return SAGIPS_OK;
}

sagips_status exchange_check(sagips_ctx* c) {
  if (!c->xs || !c->xs->err) return SAGIPS_OK;
  unsigned int e = 0;
  if (cudaMemcpy(&e, c->xs->err, sizeof e, cudaMemcpyDeviceToHost) != cudaSuccess) return SAGIPS_ERR_CUDA;
  return err_status(c, e);
}

// non-blocking: an exchange error already raised by a finished wait
sagips_status exchange_poll(sagips_ctx* c) {
  if (!c->xs || !c->xs->herr) return SAGIPS_OK;
  return err_status(c, *reinterpret_cast<volatile unsigned int*>(c->xs->herr));
}

void exchange_destroy(sagips_ctx* c) {
  ExchangeState* x = c->xs;
  if (!x) return;
  // the caller quiesces the ranks first (include/sagips.h: sagips_destroy)
  cudaDeviceSynchronize();
  for (int q = 0; q < c->cfg.world; ++q)
    if (x->peer_base[q] && q != c->cfg.rank && !x->local_peers) cudaIpcCloseMemHandle(x->peer_base[q]);
  if (x->comm_ring) ncclCommDestroy(x->comm_ring);
  if (x->comm_main) ncclCommDestroy(x->comm_main);
  cudaFree(x->win);
  cudaFree(x->gather[0]);
  cudaFree(x->gather[1]);
  cudaFree(x->outer_buf);
  if (x->one) cudaFree(x->one);
  cudaFree(x->err);
  if (x->herr) cudaFreeHost(x->herr);
  cudaFree(x->ticket);
  for (int i = 0; i < 2; ++i) {
    if (x->ev_ready[i]) cudaEventDestroy(x->ev_ready[i]);
    if (x->ev_done[i]) cudaEventDestroy(x->ev_done[i]);
  }
  if (x->side) cudaStreamDestroy(x->side);
  delete x;
  c->xs = nullptr;
}

static unsigned long long timeout_ns(const sagips_ctx* c) {
  return (unsigned long long)c->cfg.exchange_timeout_ms * 1000000ull;
}

// the two-sided pass-along ring of one version over the inner group (side stream)
static sagips_status nccl_ring(sagips_ctx* c, uint64_t step) {
  ExchangeState* x = c->xs;
  const size_t pw = slot_floats(c);
  float* gbuf = x->gather[step & 1];
  for (int j = 1; j < x->g; ++j) {
    const int send_pos = (x->pos - j + 1 + x->g) % x->g;
    const int recv_pos = (x->pos - j + x->g) % x->g;
    NCK(ncclGroupStart());
    NCK(ncclSend(gbuf + send_pos * slot_stride(c), pw, ncclFloat32, x->succ, x->comm_ring, x->side));
    NCK(ncclRecv(gbuf + recv_pos * slot_stride(c), pw, ncclFloat32, x->pred, x->comm_ring, x->side));
    NCK(ncclGroupEnd());
  }
  return SAGIPS_OK;
}

// one-sided store of `src` (pw floats) into slot [origin = this rank][version]
// of each destination's window, then its tag := version + 1 (release)
static sagips_status push_to(sagips_ctx* c, const float* src, const int* dst_ranks, int ndst, uint64_t version,
                             cudaStream_t st) {
  ExchangeState* x = c->xs;
  PushAllArgs pa{};
  for (int j = 0; j < ndst; ++j) {
    char* db = x->peer_base[dst_ranks[j]];
    pa.dst[j] = slot_ptr(db, c, c->cfg.rank, version);
    pa.dst_flag[j] = &flags_ptr(db, c)->tag[c->cfg.rank][version % kVersions];
    pa.off[j] = 0;
    pa.len[j] = (int64_t)slot_floats(c);
  }
  k_push<<<dim3(push_ctas((int64_t)slot_floats(c)), ndst), 256, 0, st>>>(src, (int64_t)slot_floats(c), pa, version + 1,
                                                                       x->ticket);
  count_launch();
  return SAGIPS_OK;
}

sagips_status exchange_push(sagips_ctx* c, uint64_t step, cudaStream_t st) {
  const auto& g = c->cfg;
  if (g.world == 1 || g.mode == SAGIPS_MODE_NONE || g.mode == SAGIPS_MODE_SYNC_ALLREDUCE) return SAGIPS_OK;
  sagips_status s = ensure_state(c);
  if (s != SAGIPS_OK) return s;
  ExchangeState* x = c->xs;
  const size_t pw = slot_floats(c);
  if (x->g == 1) return SAGIPS_OK;
  if (one_sided(c)) {
    if (!x->peers_ok) { c->err = "sagips_connect_peers not called"; return SAGIPS_ERR_STATE; }
    int dst[kMaxWorld];
    if (g.mode == SAGIPS_MODE_RMA_CHUNKED) {
      // reduce-scatter: chunk q of the packet into member q's window (slot origin = me, version t)
      const int64_t cs = chunk_floats(c, x->g), n = (int64_t)slot_floats(c);
      PushAllArgs pa{};
      int nd = 0;
      for (int q = 0; q < x->g; ++q) {
        if (q == x->pos) continue;
        char* db = x->peer_base[x->first + q];
        const int64_t off = std::min(n, q * cs), len = std::min(n, (q + 1) * cs) - off;
        pa.dst[nd] = slot_ptr(db, c, g.rank, step) + off;
        pa.dst_flag[nd] = &flags_ptr(db, c)->tag[g.rank][step % kVersions];
        pa.off[nd] = off;
        pa.len[nd] = len;
        ++nd;
      }
      k_push<<<dim3(push_ctas(cs), nd), 256, 0, st>>>(c->g_dW, 0, pa, step + 1, x->ticket);
      count_launch();
      return SAGIPS_OK;
    }
    if (g.mode == SAGIPS_MODE_RMA_ALLGATHER) {
      for (int j = 1; j < x->g; ++j) dst[j - 1] = x->first + (x->pos + j) % x->g;  // pos+1, pos+2, ...
      return push_to(c, c->g_dW, dst, x->g - 1, step, st);
    }
    dst[0] = x->succ;
    s = push_to(c, c->g_dW, dst, 1, step, st);
    if (s != SAGIPS_OK) return s;
    if (x->g > 2) {
      // the agent forwards origins pos-1 .. pos-(g-2) of this version
      char* sb = x->peer_base[x->succ];
      XCK(cudaEventRecord(x->ev_ready[step & 1], st));
      XCK(cudaStreamWaitEvent(x->side, x->ev_ready[step & 1], 0));
      FwdArgs a{};
      a.hops = x->g - 2;
      char* own = x->peer_base[g.rank];
      for (int j = 1; j <= x->g - 2; ++j) {
        const int o = x->first + (x->pos - j + x->g) % x->g;
        a.src[j - 1] = slot_ptr(own, c, o, step);
        a.src_flag[j - 1] = &flags_ptr(own, c)->tag[o][step % kVersions];
        a.dst[j - 1] = slot_ptr(sb, c, o, step);
        a.dst_flag[j - 1] = &flags_ptr(sb, c)->tag[o][step % kVersions];
      }
      k_forward<<<1, 1024, 0, x->side>>>(a, (int64_t)pw, step + 1, timeout_ns(c), err_words(x));
      count_launch();
    }
  } else {
    if (!x->comm_ring) { c->err = "sagips_connect_nccl not called"; return SAGIPS_ERR_STATE; }
    float* gbuf = x->gather[step & 1];
    XCK(cudaMemcpyAsync(gbuf + x->pos * slot_stride(c), c->g_dW, sizeof(float) * pw, cudaMemcpyDeviceToDevice, st));
    XCK(cudaEventRecord(x->ev_ready[step & 1], st));
    XCK(cudaStreamWaitEvent(x->side, x->ev_ready[step & 1], 0));
    s = nccl_ring(c, step);
    if (s != SAGIPS_OK) return s;
    XCK(cudaEventRecord(x->ev_done[step & 1], x->side));
    x->ring_issued[step & 1] = true;
    x->ring_step[step & 1] = step;
  }
  return SAGIPS_OK;
}

// the leaders' outer ring runs after step `step`'s inner fold on this rank
static bool outer_fires(const sagips_ctx* c, uint64_t step) {
  const auto& g = c->cfg;
  if (g.mode == SAGIPS_MODE_ARAR || n_leaders(g) < 2 || g.outer_every <= 0) return false;
  if ((step + 1) % (uint64_t)g.outer_every != 0) return false;
  return is_leader(g);  // leaders only
}

// the two-sided outer ring (ARAR among the leaders): pass-along
// over NCCL send/recv, then the ascending fold into `reduced` (no Adam)
static sagips_status outer_ring_nccl(sagips_ctx* c, cudaStream_t st) {
  ExchangeState* x = c->xs;
  const auto& g = c->cfg;
  const int nlead = x->nlead;
  if (!x->comm_main) { c->err = "sagips_connect_nccl not called (outer ring)"; return SAGIPS_ERR_STATE; }
  const size_t pw = slot_floats(c);
  const int lp = g.rank / g.group_size;
  const int lsucc = ((lp + 1) % nlead) * g.group_size, lpred = ((lp + nlead - 1) % nlead) * g.group_size;
  const size_t ps = slot_stride(c);
  XCK(cudaMemcpyAsync(x->outer_buf + lp * ps, c->reduced, sizeof(float) * pw, cudaMemcpyDeviceToDevice, st));
  for (int j = 1; j < nlead; ++j) {
    const int sp = (lp - j + 1 + nlead) % nlead, rp = (lp - j + nlead) % nlead;
    NCK(ncclGroupStart());
    NCK(ncclSend(x->outer_buf + sp * ps, pw, ncclFloat32, lsucc, x->comm_main, st));
    NCK(ncclRecv(x->outer_buf + rp * ps, pw, ncclFloat32, lpred, x->comm_main, st));
    NCK(ncclGroupEnd());
  }
  PacketList pl{};
  pl.count = nlead;
  for (int i = 0; i < nlead; ++i) pl.p[i] = x->outer_buf + i * ps;
  launch_fold(pl, (int64_t)pw, c->reduced, g.reduce_mean ? (float)nlead : 1.0f, st);
  return SAGIPS_OK;
}

// A step can be captured into a CUDA graph unless it depends on work recorded
// outside the capture: the two-sided rings wait, in pull(t), for the side
// stream's NCCL ring of an earlier step.  The one-sided ring's forwarding
// agent (side stream) is joined back into the step stream at the end of the
// captured step (exchange_join).
// steps whose outer ring fires on this rank run eagerly: their launch
// sequence differs, and alternating topologies would re-instantiate the
// executable graph twice per outer period (measured: 3.71 vs 2.65 ms per
// step at N = 4, g = 2, h = 10)
bool exchange_outer_step(const sagips_ctx* c, uint64_t step) { return c->cfg.world > 1 && outer_fires(c, step); }
bool exchange_graph_ok(const sagips_ctx* c) {
  const auto& g = c->cfg;
  if (g.world == 1 || g.mode == SAGIPS_MODE_NONE || g.mode == SAGIPS_MODE_SYNC_ALLREDUCE) return true;
  return one_sided(c);
}
sagips_status exchange_join(sagips_ctx* c, cudaStream_t st) {
  ExchangeState* x = c->xs;
  if (!x || !one_sided(c) || c->cfg.mode != SAGIPS_MODE_RMA_ARAR_ARAR || x->g <= 2) return SAGIPS_OK;
  XCK(cudaEventRecord(x->ev_done[0], x->side));
  XCK(cudaStreamWaitEvent(st, x->ev_done[0], 0));
  return SAGIPS_OK;
}

// pull(t) applies Adam(G) itself (k_fold_adam) for the one-sided modes
bool exchange_fuses_adam(const sagips_ctx* c, uint64_t step) {
  (void)step;
  const auto& g = c->cfg;
  if (g.world == 1 || g.mode == SAGIPS_MODE_NONE) return true;  // no exchange: copy + Adam(G) in one kernel
  return g.world > 1 && one_sided(c) && c->xs && (c->xs->g > 1 || outer_one_sided(c)) && c->xs->peers_ok;
}

// one-sided pull (modes RMA_ARAR_ARAR, RMA_ALLGATHER): k_wait on the inner
// tags of version t - s, k_fold_adam (ascending fold, Adam(G) unless the
// outer ring fires or adam == NULL); when the outer ring fires on this
// leader: the inner sum goes to the other leaders (one-sided, or NCCL) and
// their ascending fold is applied.
static sagips_status pull_one_sided(sagips_ctx* c, uint64_t step, cudaStream_t st, const GenAdam* adam) {
  ExchangeState* x = c->xs;
  const auto& g = c->cfg;
  const size_t pw = slot_floats(c);
  const int64_t stale = (int64_t)step - g.staleness;  // version of the others' packets
  char* own = x->peer_base[g.rank];
  const bool outer = outer_fires(c, step);
  FoldAdamArgs f{};
  f.reduced = c->reduced;
  f.pw = (int64_t)pw;
  f.divisor = g.reduce_mean ? (float)x->g : 1.0f;
  f.err = x->err;
  if (g.mode == SAGIPS_MODE_RMA_CHUNKED && x->g > 1) {
    // 1. the other members' chunk `pos` of version t in the own window
    const int64_t cs = chunk_floats(c, x->g), n = (int64_t)pw;
    const uint64_t vag = step + 2;  // the all-gather's slots: version t + 2 (free while staleness is 0)
    WaitArgs w{};
    w.count = x->g - 1;
    for (int j = 1; j < x->g; ++j) {
      const int o = x->first + (x->pos - j + x->g) % x->g;
      w.flag[j - 1] = &flags_ptr(own, c)->tag[o][step % kVersions];
      w.want[j - 1] = (unsigned long long)step + 1;
    }
    k_wait<<<1, 32, 0, st>>>(w, timeout_ns(c), err_words(x), reinterpret_cast<unsigned long long*>(&c->stats->wait_ns),
                             &c->stats->outer_fired);
    count_launch();
    // 2. fold chunk `pos` (ascending origins) into every member's window
    RsArgs ra{};
    ra.pl.count = x->g;
    for (int q = 0; q < x->g; ++q) {
      const int o = x->first + q;
      ra.pl.p[q] = (o == g.rank) ? c->g_dW : slot_ptr(own, c, o, step);
    }
    ra.ndst = 0;
    ra.dst[ra.ndst++] = slot_ptr(own, c, g.rank, vag);
    for (int q = 0; q < x->g; ++q) {
      if (q == x->pos) continue;
      char* db = x->peer_base[x->first + q];
      ra.dst[ra.ndst] = slot_ptr(db, c, g.rank, vag);
      ra.flag[ra.ndst] = &flags_ptr(db, c)->tag_ag[g.rank][vag % kVersions];
      ++ra.ndst;
    }
    ra.off = std::min(n, x->pos * cs);
    ra.len = std::min(n, (x->pos + 1) * cs) - ra.off;
    ra.divisor = f.divisor;
    ra.tag = (unsigned long long)step + 1;
    ra.ticket = x->ticket + (kMaxWorld - 1);
    ra.err = x->err;
    {
      bool vec = true;
      for (int q = 0; q < ra.pl.count; ++q) vec = vec && (reinterpret_cast<uintptr_t>(ra.pl.p[q]) & 15u) == 0;
      for (int d = 0; d < ra.ndst; ++d) vec = vec && (reinterpret_cast<uintptr_t>(ra.dst[d]) & 15u) == 0;
      ra.vec = (vec && ra.len >= (int64_t(1) << 18)) ? 1 : 0;
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>((ra.len / (ra.vec ? 4 : 1) + 255) / 256, 592)));
      lc.blockDim = dim3(256);
      lc.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      XCK(cudaLaunchKernelEx(&lc, k_rs_fold, ra));
      count_launch();
    }
    // 3. the other members' reduced chunks
    WaitArgs w2{};
    w2.count = x->g - 1;
    for (int j = 1; j < x->g; ++j) {
      const int o = x->first + (x->pos - j + x->g) % x->g;
      w2.flag[j - 1] = &flags_ptr(own, c)->tag_ag[o][vag % kVersions];
      w2.want[j - 1] = (unsigned long long)step + 1;
    }
    k_wait<<<1, 32, 0, st>>>(w2, timeout_ns(c), err_words(x), nullptr, nullptr);
    count_launch();
    // 4. gather the chunks (+ Adam(G) below)
    f.pl.count = x->g;
    for (int q = 0; q < x->g; ++q) f.pl.p[q] = slot_ptr(own, c, x->first + q, vag);
    f.gather_chunk = cs;
  } else if (stale >= 0) {
    WaitArgs w{};
    w.count = x->g - 1;
    for (int j = 1; j < x->g; ++j) {
      const int o = x->first + (x->pos - j + x->g) % x->g;
      w.flag[j - 1] = &flags_ptr(own, c)->tag[o][stale % kVersions];
      w.want[j - 1] = (unsigned long long)stale + 1;
    }
    k_wait<<<1, 32, 0, st>>>(w, timeout_ns(c), err_words(x), reinterpret_cast<unsigned long long*>(&c->stats->wait_ns),
                             &c->stats->outer_fired);
    count_launch();
    f.pl.count = x->g;
    for (int i = 0; i < x->g; ++i) {
      const int o = x->first + i;
      f.pl.p[i] = (o == g.rank) ? c->g_dW : slot_ptr(own, c, o, stale);
    }
  } else {
    // before step s the other members' packets are zero (R12): own packet only
    XCK(cudaMemsetAsync(&c->stats->outer_fired, 0, sizeof(uint32_t), st));
    f.pl.count = 1;
    f.pl.p[0] = c->g_dW;
  }
  if (adam && !outer) {
    f.do_adam = 1;
    f.a = *adam;
  }
  XCK(launch_fold_adam(f, st));
  if (!outer) return SAGIPS_OK;
  // the outer ring of the leaders (R13): fold of the leaders' inner sums of step t
  FoldAdamArgs o{};
  o.reduced = c->reduced;
  o.pw = (int64_t)pw;
  o.err = x->err;
  if (adam) {
    o.do_adam = 1;
    o.a = *adam;
  }
  if (outer_one_sided(c)) {
    int dst[kMaxWorld], nd = 0;
    for (int l = 0; l < x->nlead; ++l)
      if (l * g.group_size != g.rank) dst[nd++] = l * g.group_size;
    sagips_status s = push_to(c, c->reduced, dst, nd, step, st);
    if (s != SAGIPS_OK) return s;
    WaitArgs w{};
    w.count = nd;
    for (int j = 0; j < nd; ++j) {
      w.flag[j] = &flags_ptr(own, c)->tag[dst[j]][step % kVersions];
      w.want[j] = (unsigned long long)step + 1;
    }
    k_wait<<<1, 32, 0, st>>>(w, timeout_ns(c), err_words(x), nullptr, nullptr);
    count_launch();
    o.pl.count = x->nlead;
    for (int l = 0; l < x->nlead; ++l) {
      const int r = l * g.group_size;
      o.pl.p[l] = (r == g.rank) ? c->reduced : slot_ptr(own, c, r, step);
    }
    o.divisor = g.reduce_mean ? (float)x->nlead : 1.0f;
  } else {
    sagips_status s = outer_ring_nccl(c, st);
    if (s != SAGIPS_OK) return s;
    o.pl.count = 1;  // Adam(G) on the folded outer sum (identity fold, gated by err)
    o.pl.p[0] = c->reduced;
    o.divisor = 1.0f;
  }
  XCK(launch_fold_adam(o, st));
  XCK(cudaMemcpyAsync(&c->stats->outer_fired, x->one, sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
  return SAGIPS_OK;
}

sagips_status exchange_pull(sagips_ctx* c, uint64_t step, cudaStream_t st, const GenAdam* adam) {
  const auto& g = c->cfg;
  const size_t pw = slot_floats(c);
  if (adam && !exchange_fuses_adam(c, step)) {
    c->err = "exchange_pull: fused Adam(G) requested where it does not apply";
    return SAGIPS_ERR_STATE;
  }
  if (g.world == 1 || g.mode == SAGIPS_MODE_NONE) {
    if (adam) {  // the "reduced" packet is the own one: one launch copies it and applies Adam(G)
      FoldAdamArgs f{};
      f.pl.count = 1;
      f.pl.p[0] = c->g_dW;
      f.reduced = c->reduced;
      f.pw = (int64_t)pw;
      f.divisor = 1.0f;
      f.do_adam = 1;
      f.a = *adam;
      f.zero_word = &c->stats->outer_fired;
      XCK(launch_fold_adam(f, st));
      return SAGIPS_OK;
    }
    XCK(cudaMemsetAsync(&c->stats->outer_fired, 0, sizeof(uint32_t), st));
    XCK(cudaMemcpyAsync(c->reduced, c->g_dW, sizeof(float) * pw, cudaMemcpyDeviceToDevice, st));
    return SAGIPS_OK;
  }
  sagips_status s = ensure_state(c);
  if (s != SAGIPS_OK) return s;
  ExchangeState* x = c->xs;
  if (one_sided(c) && (x->g > 1 || outer_one_sided(c))) {
    if (!x->peers_ok) { c->err = "sagips_connect_peers not called"; return SAGIPS_ERR_STATE; }
    return pull_one_sided(c, step, st, adam);
  }
  XCK(cudaMemsetAsync(&c->stats->outer_fired, 0, sizeof(uint32_t), st));
  if (g.mode == SAGIPS_MODE_SYNC_ALLREDUCE) {
    if (!x->comm_main) { c->err = "sagips_connect_nccl not called"; return SAGIPS_ERR_STATE; }
    NCK(ncclAllReduce(c->g_dW, c->reduced, pw, ncclFloat32, ncclSum, x->comm_main, st));
    if (g.reduce_mean) {
      PacketList pl{};
      pl.count = 1;
      pl.p[0] = c->reduced;
      launch_fold(pl, (int64_t)pw, c->reduced, (float)g.world, st);
    }
    return SAGIPS_OK;
  }
  const int64_t stale = (int64_t)step - g.staleness;  // version of the others' packets
  PacketList pl{};
  pl.count = x->g;
  if (x->g == 1) {
    pl.p[0] = c->g_dW;
  } else {
    if (stale >= 0) {
      const int v = (int)(stale & 1);
      if (!x->ring_issued[v] || x->ring_step[v] != (uint64_t)stale) {
        c->err = "pull: ring of the needed version was not issued";
        return SAGIPS_ERR_STATE;
      }
      XCK(cudaStreamWaitEvent(st, x->ev_done[v], 0));
    }
    for (int i = 0; i < x->g; ++i)
      pl.p[i] = (i == x->pos) ? c->g_dW : (stale >= 0 ? x->gather[stale & 1] + i * slot_stride(c) : nullptr);
  }
  if (stale < 0 && x->g > 1) {
    PacketList ownp{};
    ownp.count = 1;
    ownp.p[0] = c->g_dW;
    launch_fold(ownp, (int64_t)pw, c->reduced, g.reduce_mean ? (float)x->g : 1.0f, st);
  } else {
    launch_fold(pl, (int64_t)pw, c->reduced, g.reduce_mean ? (float)x->g : 1.0f, st);
  }
  if (!outer_fires(c, step)) return SAGIPS_OK;
  s = outer_ring_nccl(c, st);
  if (s != SAGIPS_OK) return s;
  XCK(cudaMemcpyAsync(&c->stats->outer_fired, x->one, sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
  return SAGIPS_OK;
}

}  // namespace sagips

using namespace sagips;

extern "C" {

sagips_status sagips_ipc_handle(sagips_ctx* c, void* host_handle, size_t bytes) {
  if (!c || !host_handle || bytes != SAGIPS_IPC_HANDLE_BYTES) return SAGIPS_ERR_INVALID_ARG;
  std::memset(host_handle, 0, bytes);
  if (!one_sided(c) || c->cfg.world == 1) return SAGIPS_OK;  // nothing to share
  sagips_status s = ensure_state(c);
  if (s != SAGIPS_OK) return s;
  static_assert(sizeof(cudaIpcMemHandle_t) == SAGIPS_IPC_HANDLE_BYTES, "handle size");
  std::memcpy(host_handle, &c->xs->handle, bytes);
  return SAGIPS_OK;
}

sagips_status sagips_connect_peers(sagips_ctx* c, const void* host_handles, size_t bytes) {
  if (!c || !host_handles || bytes != (size_t)SAGIPS_IPC_HANDLE_BYTES * c->cfg.world) return SAGIPS_ERR_INVALID_ARG;
  if (!one_sided(c) || c->cfg.world == 1) return SAGIPS_OK;
  sagips_status s = ensure_state(c);
  if (s != SAGIPS_OK) return s;
  ExchangeState* x = c->xs;
  if (x->peers_ok) { c->err = "peers already connected"; return SAGIPS_ERR_STATE; }
  const char* h = (const char*)host_handles;
  for (int q = 0; q < c->cfg.world; ++q) {
    if (!maps_peer(c, q)) continue;
    if (q == c->cfg.rank) {
      x->peer_base[q] = reinterpret_cast<char*>(x->win);
      continue;
    }
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, h + (size_t)q * SAGIPS_IPC_HANDLE_BYTES, sizeof hd);
    void* p = nullptr;
    XCK(cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess));
    x->peer_base[q] = reinterpret_cast<char*>(p);
  }
  x->peers_ok = true;
  return SAGIPS_OK;
}

sagips_status sagips_window_ptr(sagips_ctx* c, uint64_t* dev_ptr) {
  if (!c || !dev_ptr) return SAGIPS_ERR_INVALID_ARG;
  *dev_ptr = 0;
  if (!one_sided(c) || c->cfg.world == 1) return SAGIPS_OK;
  sagips_status s = ensure_state(c);
  if (s != SAGIPS_OK) return s;
  *dev_ptr = (uint64_t)(uintptr_t)c->xs->win;
  return SAGIPS_OK;
}

sagips_status sagips_connect_peers_local(sagips_ctx* c, const uint64_t* dev_ptrs, size_t n) {
  if (!c || !dev_ptrs || n != (size_t)c->cfg.world) return SAGIPS_ERR_INVALID_ARG;
  if (!one_sided(c) || c->cfg.world == 1) return SAGIPS_OK;
  sagips_status s = ensure_state(c);
  if (s != SAGIPS_OK) return s;
  ExchangeState* x = c->xs;
  if (x->peers_ok) { c->err = "peers already connected"; return SAGIPS_ERR_STATE; }
  if (dev_ptrs[c->cfg.rank] != (uint64_t)(uintptr_t)x->win) { c->err = "own window pointer mismatch"; return SAGIPS_ERR_INVALID_ARG; }
  for (int q = 0; q < c->cfg.world; ++q) {
    if (!maps_peer(c, q)) continue;
    if (!dev_ptrs[q]) { c->err = "null peer window"; return SAGIPS_ERR_INVALID_ARG; }
    x->peer_base[q] = reinterpret_cast<char*>((uintptr_t)dev_ptrs[q]);
  }
  x->local_peers = true;
  x->peers_ok = true;
  return SAGIPS_OK;
}

sagips_status sagips_nccl_unique_id(void* host_id, size_t bytes) {
  if (!host_id || bytes != SAGIPS_NCCL_ID_BYTES) return SAGIPS_ERR_INVALID_ARG;
  static_assert(sizeof(ncclUniqueId) == SAGIPS_NCCL_ID_BYTES, "nccl id size");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return SAGIPS_ERR_CUDA;
  std::memcpy(host_id, &id, bytes);
  return SAGIPS_OK;
}

sagips_status sagips_connect_nccl(sagips_ctx* c, const void* host_id, size_t bytes) {
  if (!c || !host_id || bytes != SAGIPS_NCCL_ID_BYTES) return SAGIPS_ERR_INVALID_ARG;
  if (!needs_nccl(c)) return SAGIPS_OK;
  sagips_status s = ensure_state(c);
  if (s != SAGIPS_OK) return s;
  ExchangeState* x = c->xs;
  ncclUniqueId id;
  std::memcpy(&id, host_id, sizeof id);
  NCK(ncclCommInitRank(&x->comm_main, c->cfg.world, id, c->cfg.rank));
  NCK(ncclCommSplit(x->comm_main, 0, c->cfg.rank, &x->comm_ring, nullptr));
  // NCCL sets up peer connections lazily, on the first send/recv between two
  // ranks (hundreds of ms): exercise the leaders' outer ring and the inner
  // two-sided ring here, so no training step pays for it
  const auto& g = c->cfg;
  const int nlead = x->nlead;
  float* tmp = nullptr;
  XCK(cudaMalloc(&tmp, 2 * sizeof(float)));
  if (nlead >= 2 && g.outer_every > 0 && is_leader(g)) {
    const int lp = g.rank / g.group_size;
    NCK(ncclGroupStart());
    NCK(ncclSend(tmp, 1, ncclFloat32, ((lp + 1) % nlead) * g.group_size, x->comm_main, x->side));
    NCK(ncclRecv(tmp + 1, 1, ncclFloat32, ((lp + nlead - 1) % nlead) * g.group_size, x->comm_main, x->side));
    NCK(ncclGroupEnd());
  }
  if (x->g > 1 && !one_sided(c)) {
    NCK(ncclGroupStart());
    NCK(ncclSend(tmp, 1, ncclFloat32, x->succ, x->comm_ring, x->side));
    NCK(ncclRecv(tmp + 1, 1, ncclFloat32, x->pred, x->comm_ring, x->side));
    NCK(ncclGroupEnd());
  }
  XCK(cudaStreamSynchronize(x->side));
  XCK(cudaFree(tmp));
  return SAGIPS_OK;
}

}  // extern "C"
