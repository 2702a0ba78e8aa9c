// Multi-color tree allreduce over NVLink/NVSwitch peer memory (sm_100a).
//
// Reference semantics (/root/reference/pkg/src/minidist/collectives.py):
//   * allreduce_multicolor (:225-268): the payload is split into k contiguous
//     chunks (make_chunk_plan, topology.py:103-120); chunk c is reduced up
//     color tree c -- every node folds, IN CHILD-LIST ORDER, its own value and
//     its children's subtree sums (_tree_up_task, :271-286) -- and the root's
//     result is broadcast back down the same tree (_tree_down_task, :289-296).
//   * allreduce_ring (:302-359) is the same fold on a chain (each node folds
//     its successor), reduce_then_broadcast (:365-409) a star whose root folds
//     every rank in ascending rank order. All three are one kernel here; the
//     fold tree is data (md_plan_t).
//
// B200 design: ONE persistent kernel per call and rank, picked per call
// (md_allreduce_ex; md_plan_set_route pins one): LL push, one-shot pull,
// owner-push (plain calls and the sharded SGD update), the tiled all-pull
// stream kernel, the channelized tree and the work-queue tree. The tree
// kernels move each color's chunk along its tree (UP folds in the reference
// order with __fadd_rn, DOWN copies the parent's final); the others evaluate
// each color's fold program (the same adds in the same order) on data pulled
// or pushed over NVLink. The optional prologue folds per-worker gradient
// buffers (sgd.py:335-353) into the own value, and the optional epilogue
// applies the SGD (momentum / weight-decay) update as soon as a segment's
// sum is final, so the gradient is never re-read from HBM.
//
// Synchronisation (replaces the transport's expose/pull and the length-header
// barrier of _check_same_length, :157-174): epoch-tagged flags in peer-mapped
// control blocks, polled with ld.acquire.sys (published as described at
// publish_flags); an entry barrier carries every rank's
// buffer length (LengthMismatch) and route word (InvalidConfig) and an exit
// barrier guarantees no peer still reads a buffer when the call returns.
// Waits are bounded by a globaltimer watchdog (NotExposed). No flag is ever
// reset: epochs only grow.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include "md_common.cuh"

namespace md {

constexpr int kMaxSegs = 4096;        // per color
constexpr int kLLElems = 262144;      // LL inbox: payload floats per (parity, source)
constexpr int kMaxTiles = 65536;      // stream kernel: tiles per call
constexpr int kArThreads = 512;
// float4 per thread per source per pass: 512 threads x 2 x 16 B keeps >= 16 KB
// per SM in flight per source (NVLink needs ~5 KB/SM at 775 GB/s x 1 us)
constexpr int kUnroll = 2;

struct Ctrl {
  unsigned long long arrive_len[MD_MAX_RANKS];  // from peer r: n | n_workers << 56
  unsigned long long arrive_cfg[MD_MAX_RANKS];  // from peer r: its route word (cfg_word)
  uint32_t arrive_epoch[MD_MAX_RANKS];
  uint32_t done_epoch[MD_MAX_RANKS];
  uint32_t pad0[32 - 2 * MD_MAX_RANKS % 32];
  uint32_t queue_head;   // local work queue counter
  uint32_t pad1[31];
  uint32_t finished;     // CTAs of this rank done with the current call
  uint32_t abort_flag;   // set by any CTA of this rank that bailed out
  uint32_t epoch;        // calls completed by this rank (device-side counter)
  uint32_t finished2;    // one-shot kernel: CTAs of this rank done with their stores
  uint32_t pad2[28];
  uint32_t up[MD_MAX_COLORS][MD_MAX_RANKS + 1][kMaxSegs];
  uint32_t down[MD_MAX_COLORS][kMaxSegs];
  // LL inbox (allreduce_ll_kernel): source r pushes (value bits | epoch << 32)
  // words for call `epoch` into ll[epoch & 1][r]; the epoch tag makes every
  // 8-byte word self-validating, so no flag or fence orders the data.
  unsigned long long ll[2][MD_MAX_RANKS][kLLElems];
  // stream kernel: rd[r][t] = epoch once rank r has finished reading tile t of
  // this rank's buffer (then the tile may be overwritten with the result)
  uint32_t rd[MD_MAX_RANKS][kMaxTiles];
};

struct Task {
  int32_t type;  // 0 = UP (fold), 1 = DOWN (copy final from parent),
                 // 2 = OWNER (fold every rank's value with the element's color program)
  int32_t color;
  int32_t stage;
  int32_t n_fold;
  int32_t parent;   // -1 at the root
  int32_t my_slot;  // UP, non-root: my position in the parent's fold list
  int32_t n_down;   // ranks that need my final value (children)
  int32_t is_leaf;
  int32_t fold_src[MD_MAX_RANKS + 1];
  int32_t fold_leaf[MD_MAX_RANKS + 1];
  int32_t down[MD_MAX_RANKS];
};

struct RankPlan {
  int32_t n_tasks;
  int32_t pad[3];
  Task t[2 * MD_MAX_COLORS];
};

// The whole fold of one color as a straight-line program over rank slots:
// ops in post-order (children before parents); op j overwrites slot
// op_dst[j] (the folding rank) with the left fold of the slots
// items[off_j .. off_j + op_cnt[j]) -- the rank's fold list in the reference's
// order (its own value is its own slot, a child's subtree sum is the child's
// slot, already overwritten). The color's value ends in slot `root`.
struct ColorProg {
  uint8_t n_ops, root, pad[2];
  uint8_t op_dst[MD_MAX_RANKS];
  uint8_t op_cnt[MD_MAX_RANKS];
  uint8_t items[2 * MD_MAX_RANKS];
};
struct FoldProg {
  ColorProg c[MD_MAX_COLORS];
};

struct ViewArgs {
  float* buf;
  const float* peer[MD_MAX_RANKS];
  Ctrl* ctrl;
  Ctrl* peer_ctrl[MD_MAX_RANKS];
  const float* workers[MD_MAX_WORKERS];
  float* w;
  float* mom;
  float* peer_w[MD_MAX_RANKS];  // sharded update: every rank's weights (peer-mapped)
  int32_t* err;  // host-mapped: [code, detail]
  int32_t rank;
  uint32_t epoch;
};

struct TraceEv {
  unsigned long long t;
  uint32_t cta;
  uint16_t ev, seg;
};

struct AllreduceArgs {
  const RankPlan* plan;
  int64_t n;
  int64_t seg;
  int64_t update_len;
  unsigned long long timeout_ns;
  int32_t n_ranks, k, n_views, ctas_per_view;
  int32_t max_nseg, n_workers;
  int32_t lag, max_stage;  // queue skew between pipeline stages (segments)
  int32_t has_update, vec_ok;
  float c, mu, wd_b;
  struct TraceEv* trace;  // nullable: per-CTA event log (MD_AR_TRACE=1)
  int32_t flag_gpu_fence;  // publish with fence.acq_rel.gpu + relaxed sys stores (publish_flags)
  int32_t reverse_local;   // local-only tasks walk their segments last-first
  const FoldProg* prog;    // every color's fold program (one-shot / LL / stream / owner)
  int32_t prog_k;          // colors of the fold programs (the plan's k; a.k counts owner slices)
  int32_t sharded;         // push kernel: sharded SGD update (W' pushed, momentum sharded)
  int32_t exit_sys_release;  // done flags certify REMOTE writes (owner-push): release at sys scope
  // route word every rank publishes at the entry barrier: ranks that picked a
  // different kernel / tile / segment / schedule / update mode fail together
  // with InvalidConfig instead of exchanging differently-shaped flags
  unsigned long long cfg_word;
  ViewArgs v[MD_MAX_RANKS];
};

}  // namespace md

struct md_comm {
  int32_t rank, n_ranks, device;
  md::Ctrl* ctrl;
  md::Ctrl* peer_ctrl[MD_MAX_RANKS];
  int32_t* err_host;  // pinned, mapped
  int32_t* err_dev;
  uint32_t epoch;
  double timeout_s;
};

struct md_plan {
  int32_t n_ranks, k, device;
  md::RankPlan* dev;                   // n_ranks entries
  std::vector<md::RankPlan> host;
  md::FoldProg* prog_dev;              // the same trees as fold programs (one-shot kernel)
  std::vector<md::RankPlan> owner_host;  // owner-computes schedule (MD_SCHED_OWNER)
  md::RankPlan* owner_dev;
  int32_t schedule;                    // MD_SCHED_TREE / MD_SCHED_OWNER
  int32_t route;                       // MD_ROUTE_* (md_plan_set_route; AUTO = by size)
  int64_t tile;                        // tile override of the tiled routes (0 = auto)
};

namespace md {

// ---- chunk / segment geometry (make_chunk_plan, topology.py:103-120) --------
__host__ __device__ __forceinline__ void chunk_of(int64_t n, int k, int c, int64_t* start,
                                                  int64_t* len) {
  int64_t base = n / k, extra = n % k;
  *start = c * base + (c < extra ? c : extra);
  *len = base + (c < extra ? 1 : 0);
}
__host__ __device__ __forceinline__ int64_t nseg_of(int64_t start, int64_t len, int64_t seg) {
  if (len <= 0) return 0;
  int64_t a = start & ~int64_t(3);
  return (start + len - a + seg - 1) / seg;
}

// ---- fold programs (ColorProg): a color's whole fold over rank slots ----------
__device__ __forceinline__ int color_of(int64_t n, int k, int64_t i) {
  const int64_t base = n / k, extra = n % k;
  const int64_t big = (base + 1) * extra;  // the first `extra` chunks hold base + 1
  if (i < big) return static_cast<int>(i / (base + 1));
  return static_cast<int>(extra + (i - big) / base);
}

__device__ __forceinline__ float fold_prog(const ColorProg& p, float* slots, int64_t E,
                                           int64_t e) {
  int off = 0;
  for (int j = 0; j < p.n_ops; ++j) {
    const int cnt = p.op_cnt[j];
    float acc = slots[p.items[off] * E + e];
    for (int q = 1; q < cnt; ++q) acc = __fadd_rn(acc, slots[p.items[off + q] * E + e]);
    slots[p.op_dst[j] * E + e] = acc;
    off += cnt;
  }
  return slots[p.root * E + e];
}

__device__ __forceinline__ float4 fold_prog4(const ColorProg& p, float* slots, int64_t E,
                                             int64_t e) {  // e: multiple of 4
  int off = 0;
  for (int j = 0; j < p.n_ops; ++j) {
    const int cnt = p.op_cnt[j];
    float4 acc = *reinterpret_cast<const float4*>(slots + p.items[off] * E + e);
    for (int q = 1; q < cnt; ++q)
      acc = add4(acc, *reinterpret_cast<const float4*>(slots + p.items[off + q] * E + e));
    *reinterpret_cast<float4*>(slots + p.op_dst[j] * E + e) = acc;
    off += cnt;
  }
  return *reinterpret_cast<const float4*>(slots + p.root * E + e);
}

// ---- device helpers -----------------------------------------------------------
__device__ __forceinline__ void raise_err(const ViewArgs& v, int code, int detail) {
  volatile int32_t* e = v.err;
  if (e[0] == 0) {
    e[1] = detail;
    e[0] = code;
  }
  atomicExch(&v.ctrl->abort_flag, 1u);
}

// Thread 0 spins until *flag >= epoch. Returns false on timeout/abort.
__device__ bool wait_flag(const ViewArgs& v, const uint32_t* flag, uint32_t epoch,
                          unsigned long long timeout_ns, int detail) {
  if (epoch_ge(ld_acquire_sys(flag), epoch)) return true;
  uint64_t t0 = globaltimer_ns();
  uint32_t spins = 0;
  while (true) {
    if (epoch_ge(ld_acquire_sys(flag), epoch)) return true;
    if ((++spins & 255) == 0) {
      if (*reinterpret_cast<volatile uint32_t*>(&v.ctrl->abort_flag)) return false;
      if (globaltimer_ns() - t0 > timeout_ns) {
        raise_err(v, MD_ERR_TIMEOUT, detail);
        return false;
      }
      __nanosleep(64);
    }
  }
}

template <bool kVec>
struct Elem;
template <>
struct Elem<true> {
  using T = float4;
  static __device__ __forceinline__ T ld(const float* p, int64_t i) {
    return *reinterpret_cast<const float4*>(p + i);
  }
  static __device__ __forceinline__ T ld_stream(const float* p, int64_t i) {
    return __ldcs(reinterpret_cast<const float4*>(p + i));
  }
  static __device__ __forceinline__ void st(float* p, int64_t i, T x) {
    *reinterpret_cast<float4*>(p + i) = x;
  }
  static __device__ __forceinline__ T add(T a, T b) { return add4(a, b); }
  static constexpr int W = 4;
};
template <>
struct Elem<false> {
  using T = float;
  static __device__ __forceinline__ T ld(const float* p, int64_t i) { return p[i]; }
  static __device__ __forceinline__ T ld_stream(const float* p, int64_t i) { return p[i]; }
  static __device__ __forceinline__ void st(float* p, int64_t i, T x) { p[i] = x; }
  static __device__ __forceinline__ T add(T a, T b) { return __fadd_rn(a, b); }
  static constexpr int W = 1;
};

// ---- SGD epilogue -------------------------------------------------------------
// kEpi: 0 none, 1 plain SGD, 2 + weight decay, 3 + momentum, 4 momentum + wd.
// A compile-time variant per item keeps the unrolled loops branch-free.
template <int kEpi>
__device__ __forceinline__ void sgd_elem(float& w, float g, float& m, const AllreduceArgs& a) {
  if constexpr (kEpi == 1) sgd1<false, false>(w, g, &m, a.c, a.mu, a.wd_b);
  if constexpr (kEpi == 2) sgd1<true, false>(w, g, &m, a.c, a.mu, a.wd_b);
  if constexpr (kEpi == 3) sgd1<false, true>(w, g, &m, a.c, a.mu, a.wd_b);
  if constexpr (kEpi == 4) sgd1<true, true>(w, g, &m, a.c, a.mu, a.wd_b);
}

template <int kEpi>
__device__ __forceinline__ void epi_scalar(const AllreduceArgs& a, const ViewArgs& v, int64_t i,
                                           float g) {
  if constexpr (kEpi == 0) return;
  if (i >= a.update_len) return;
  constexpr bool kMom = kEpi >= 3;
  float w = v.w[i];
  float m = kMom ? v.mom[i] : 0.f;
  sgd_elem<kEpi>(w, g, m, a);
  v.w[i] = w;
  if (kMom) v.mom[i] = m;
}

// One unrolled batch of a thread (elements b + u*nthr*W): all W/momentum loads
// are issued before any store, so 2*kUnroll 16-byte loads are in flight.
template <bool kVec, int kEpi>
__device__ __forceinline__ void epi_batch(const AllreduceArgs& a, const ViewArgs& v, int64_t b,
                                          int64_t hi, int nthr,
                                          const typename Elem<kVec>::T (&g)[kUnroll]) {
  if constexpr (kEpi == 0) return;
  constexpr bool kMom = kEpi >= 3;
  if constexpr (!kVec) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      int64_t i = b + static_cast<int64_t>(u) * nthr;
      if (i < hi) epi_scalar<kEpi>(a, v, i, g[u]);
    }
  } else {
    const int64_t last = b + static_cast<int64_t>(kUnroll - 1) * nthr * 4;
    if (last + 3 >= a.update_len || last >= hi) {  // ragged batch: element by element
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        int64_t i = b + static_cast<int64_t>(u) * nthr * 4;
        if (i < hi) {
          epi_scalar<kEpi>(a, v, i, g[u].x);
          epi_scalar<kEpi>(a, v, i + 1, g[u].y);
          epi_scalar<kEpi>(a, v, i + 2, g[u].z);
          epi_scalar<kEpi>(a, v, i + 3, g[u].w);
        }
      }
      return;
    }
    float4 w[kUnroll], m[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t i = b + static_cast<int64_t>(u) * nthr * 4;
      w[u] = __ldcs(reinterpret_cast<const float4*>(v.w + i));
      if constexpr (kMom) m[u] = __ldcs(reinterpret_cast<const float4*>(v.mom + i));
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      sgd_elem<kEpi>(w[u].x, g[u].x, m[u].x, a);
      sgd_elem<kEpi>(w[u].y, g[u].y, m[u].y, a);
      sgd_elem<kEpi>(w[u].z, g[u].z, m[u].z, a);
      sgd_elem<kEpi>(w[u].w, g[u].w, m[u].w, a);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t i = b + static_cast<int64_t>(u) * nthr * 4;
      __stcs(reinterpret_cast<float4*>(v.w + i), w[u]);
      if constexpr (kMom) __stcs(reinterpret_cast<float4*>(v.mom + i), m[u]);
    }
  }
}

// Own value at element i: the buffer, or the worker fold (worker order).
template <bool kVec>
__device__ __forceinline__ typename Elem<kVec>::T own_value(const AllreduceArgs& a,
                                                            const ViewArgs& v, int64_t i) {
  using E = Elem<kVec>;
  if (a.n_workers == 0) return E::ld(v.buf, i);
  typename E::T x = E::ld_stream(v.workers[0], i);
  for (int j = 1; j < a.n_workers; ++j) x = E::add(x, E::ld_stream(v.workers[j], i));
  return x;
}

// ---- TMA path: remote sources stream through a shared-memory ring -------------
// One elected thread issues cp.async.bulk copies of every remote fold source
// (children's subtree sums, or the parent's final segment) straight from the
// peers' HBM over NVLink into a kStages-deep ring; all threads fold the ring
// contents with the own value in the reference order, store, and run the SGD
// epilogue while the next chunks are in flight. Bytes in flight per SM are
// bounded by the ring (3 x 32 KB), not by registers, and the HBM epilogue
// overlaps the NVLink transfer instead of alternating with it.
constexpr int kStages = 4;
constexpr uint32_t kStageBytes = 48 * 1024;
constexpr uint32_t kRingBytes = kStages * kStageBytes;
// the stream and owner-push kernels' ring: (almost) all of the 227 KB a CTA
// may opt into (their static SMEM is ~1.4 KB). The stream kernel's N = 2
// fused calls fit two stages of <= 6656-float tiles (4 slots: 2 ranks, W,
// momentum); the owner-push kernel's sharded calls 3-4 stages of [N ranks |
// sum | W | momentum] at its ~2000-3000-float tiles
constexpr uint32_t kStreamRingBytes = 224 * 1024;

template <int kEpi>
__device__ __forceinline__ void item_tma(const AllreduceArgs& a, const ViewArgs& v, const Task& t,
                                         bool final_here, int64_t lo, int64_t hi, int nrem,
                                         char* ring, uint64_t* full, uint32_t& seq) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  // elements per remote source per stage (multiple of 4 -> 16-byte TMA sizes)
  const int64_t C = static_cast<int64_t>(kStageBytes / (4u * nrem)) & ~int64_t(3);
  const int64_t nch = (hi - lo + C - 1) / C;
  auto issue = [&](int64_t c) {  // thread 0 only
    const uint32_t g = seq + static_cast<uint32_t>(c);
    uint64_t* bar = &full[g % kStages];
    char* stage = ring + (g % kStages) * kStageBytes;
    const int64_t clo = lo + c * C;
    const uint32_t bytes = static_cast<uint32_t>((min(hi, clo + C) - clo) * 4);
    mbar_expect_tx(bar, bytes * nrem);
    if (t.type == 1) {
      tma_load_1d(stage, v.peer[t.parent] + clo, bytes, bar);
    } else {
      int q = 0;
      for (int j = 0; j < t.n_fold; ++j) {
        const int src = t.fold_src[j];
        if (src == v.rank) continue;
        tma_load_1d(stage + q * C * 4, v.peer[src] + clo, bytes, bar);
        ++q;
      }
    }
  };
  if (tid == 0) {
    fence_proxy_async_global();  // peers' flags were acquired in the generic proxy
    for (int64_t c = 0; c < nch && c < kStages; ++c) issue(c);
  }
  for (int64_t c = 0; c < nch; ++c) {
    const uint32_t g = seq + static_cast<uint32_t>(c);
    const char* stage = ring + (g % kStages) * kStageBytes;
    while (!mbar_try_wait(&full[g % kStages], (g / kStages) & 1)) {
    }
    const int64_t clo = lo + c * C;
    const int64_t chi = min(hi, clo + C);
    const int64_t n4 = (chi - clo) / 4;
    for (int64_t e0 = tid; e0 < n4; e0 += static_cast<int64_t>(kUnroll) * nthr) {
      const int64_t b = clo + 4 * e0;
      float4 acc[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t e = e0 + static_cast<int64_t>(u) * nthr;
        if (e >= n4) break;
        if (t.type == 1) {
          acc[u] = reinterpret_cast<const float4*>(stage)[e];
        } else {
          int q = 0;
          for (int j = 0; j < t.n_fold; ++j) {
            float4 x;
            if (t.fold_src[j] == v.rank) {
              x = own_value<true>(a, v, clo + 4 * e);
            } else {
              x = reinterpret_cast<const float4*>(stage + q * C * 4)[e];
              ++q;
            }
            acc[u] = (j == 0) ? x : add4(acc[u], x);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t e = e0 + static_cast<int64_t>(u) * nthr;
        if (e < n4) *reinterpret_cast<float4*>(v.buf + clo + 4 * e) = acc[u];
      }
      if (kEpi != 0 && final_here) epi_batch<true, kEpi>(a, v, b, chi, nthr, acc);
    }
    __syncthreads();  // every thread is done with this stage
    if (tid == 0 && c + kStages < nch) issue(c + kStages);
  }
  seq += static_cast<uint32_t>(nch);
}

// Epilogue pass over [lo, hi): every thread re-reads the elements it just
// stored (same mapping, so program order makes them visible; they are still
// in L2) and updates W (+ momentum). Kept out of the data pass so the fold's
// in-flight loads do not compete with the epilogue's registers.
template <bool kVec, int kEpi>
__device__ __forceinline__ void epilogue_pass(const AllreduceArgs& a, const ViewArgs& v,
                                              int64_t lo, int64_t hi, int tid, int nthr) {
  if constexpr (kEpi != 0) {
    using E = Elem<kVec>;
    constexpr int W = E::W;
    const int64_t step = static_cast<int64_t>(nthr) * W * kUnroll;
    for (int64_t b = lo + static_cast<int64_t>(tid) * W; b < hi; b += step) {
      typename E::T g[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        int64_t i = b + static_cast<int64_t>(u) * nthr * W;
        if (i < hi) g[u] = E::ld(v.buf, i);
      }
      epi_batch<kVec, kEpi>(a, v, b, hi, nthr, g);
    }
  }
}

// Lone-root SGD update over a 16-byte aligned [lo, hi): the sum is the buffer
// itself, so this is a pure HBM stream (read g, r/w W and v). Every load of an
// unrolled batch is issued before any math so each thread keeps 3 x kLoneU
// 16-byte loads in flight.
template <int kEpi>
__device__ __forceinline__ void lone_update(const AllreduceArgs& a, const ViewArgs& v, int64_t lo,
                                            int64_t hi, int tid, int nthr) {
  constexpr int kLoneU = 4;
  constexpr bool kMom = kEpi >= 3;
  const int64_t hi4 = min(hi, a.update_len & ~int64_t(3));
  const int64_t step = static_cast<int64_t>(nthr) * 4 * kLoneU;
  int64_t b = lo + static_cast<int64_t>(tid) * 4;
  for (; b + static_cast<int64_t>(kLoneU - 1) * nthr * 4 < hi4; b += step) {
    float4 g[kLoneU], w[kLoneU], m[kLoneU];
#pragma unroll
    for (int u = 0; u < kLoneU; ++u) {
      const int64_t i = b + static_cast<int64_t>(u) * nthr * 4;
      g[u] = __ldcs(reinterpret_cast<const float4*>(v.buf + i));
      w[u] = __ldcs(reinterpret_cast<const float4*>(v.w + i));
      if (kMom) m[u] = __ldcs(reinterpret_cast<const float4*>(v.mom + i));
    }
#pragma unroll
    for (int u = 0; u < kLoneU; ++u) {
      sgd_elem<kEpi>(w[u].x, g[u].x, m[u].x, a);
      sgd_elem<kEpi>(w[u].y, g[u].y, m[u].y, a);
      sgd_elem<kEpi>(w[u].z, g[u].z, m[u].z, a);
      sgd_elem<kEpi>(w[u].w, g[u].w, m[u].w, a);
    }
#pragma unroll
    for (int u = 0; u < kLoneU; ++u) {
      const int64_t i = b + static_cast<int64_t>(u) * nthr * 4;
      __stcs(reinterpret_cast<float4*>(v.w + i), w[u]);
      if (kMom) __stcs(reinterpret_cast<float4*>(v.mom + i), m[u]);
    }
  }
  // remainder of the thread's range (and anything past update_len): per vector
  for (; b < hi; b += static_cast<int64_t>(nthr) * 4) {
    const float4 g4 = *reinterpret_cast<const float4*>(v.buf + b);
    epi_scalar<kEpi>(a, v, b, g4.x);
    epi_scalar<kEpi>(a, v, b + 1, g4.y);
    epi_scalar<kEpi>(a, v, b + 2, g4.z);
    epi_scalar<kEpi>(a, v, b + 3, g4.w);
  }
}

// Data pass of one item over [lo, hi) (all W-aligned when kVec): DOWN copies
// the parent's final segment, UP folds its sources in the plan's order.
template <bool kVec>
__device__ __forceinline__ void item_data(const AllreduceArgs& a, const ViewArgs& v, const Task& t,
                                          int64_t lo, int64_t hi, int tid, int nthr) {
  using E = Elem<kVec>;
  constexpr int W = E::W;
  constexpr int kCopyUnroll = 2 * kUnroll;  // a copy holds nothing else in registers
  if (t.type == 2) {  // OWNER (edge elements only): every rank's value, color program
    for (int64_t i = lo + tid; i < hi; i += nthr) {
      float x[MD_MAX_RANKS];
      for (int r = 0; r < a.n_ranks; ++r) x[r] = r == v.rank ? v.buf[i] : v.peer[r][i];
      v.buf[i] = fold_prog(a.prog->c[color_of(a.n, a.prog_k, i)], x, 1, 0);
    }
    return;
  }
  if (t.type == 1) {  // DOWN: copy the parent's final value
    const float* src = v.peer[t.parent];
    const int64_t cstep = static_cast<int64_t>(nthr) * W * kCopyUnroll;
    for (int64_t b = lo + static_cast<int64_t>(tid) * W; b < hi; b += cstep) {
      typename E::T x[kCopyUnroll];
#pragma unroll
      for (int u = 0; u < kCopyUnroll; ++u) {
        int64_t i = b + static_cast<int64_t>(u) * nthr * W;
        if (i < hi) x[u] = E::ld(src, i);
      }
#pragma unroll
      for (int u = 0; u < kCopyUnroll; ++u) {
        int64_t i = b + static_cast<int64_t>(u) * nthr * W;
        if (i < hi) E::st(v.buf, i, x[u]);
      }
    }
    return;
  }
  if (t.n_fold == 1 && a.n_workers == 0) return;  // lone rank: the sum is the buffer
  // UP: fold own value and children in the plan's order
  const int64_t step = static_cast<int64_t>(nthr) * W * kUnroll;
  constexpr int kGroup = 4;  // fold sources whose loads are in flight together
  for (int64_t b = lo + static_cast<int64_t>(tid) * W; b < hi; b += step) {
    typename E::T acc[kUnroll];
    for (int j0 = 0; j0 < t.n_fold; j0 += kGroup) {
      typename E::T x[kGroup][kUnroll];
      // issue every load of the group first (remote latency ~2 us) ...
#pragma unroll
      for (int q = 0; q < kGroup; ++q) {
        const int j = j0 + q;
        if (j >= t.n_fold) break;
        const int src_rank = t.fold_src[j];
        const float* src = src_rank == v.rank ? nullptr : v.peer[src_rank];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          int64_t i = b + static_cast<int64_t>(u) * nthr * W;
          if (i < hi) x[q][u] = src ? E::ld(src, i) : own_value<kVec>(a, v, i);
        }
      }
      // ... then add strictly in the reference's fold order
#pragma unroll
      for (int q = 0; q < kGroup; ++q) {
        const int j = j0 + q;
        if (j >= t.n_fold) break;
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) acc[u] = (j == 0) ? x[q][u] : E::add(acc[u], x[q][u]);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      int64_t i = b + static_cast<int64_t>(u) * nthr * W;
      if (i < hi) E::st(v.buf, i, acc[u]);
    }
  }
}

// The kernel is instantiated per epilogue variant (chosen on the host for the
// whole call); the epilogue runs where an item makes a segment final.
template <bool kVec, int kEpi>
__device__ __forceinline__ void item_dispatch(const AllreduceArgs& a, const ViewArgs& v,
                                              const Task& t, bool final_here, int64_t lo,
                                              int64_t hi, int tid, int nthr) {
  item_data<kVec>(a, v, t, lo, hi, tid, nthr);
  if (kEpi != 0 && final_here) epilogue_pass<kVec, kEpi>(a, v, lo, hi, tid, nthr);
}

// ---- optional tracing: %globaltimer events, producer and consumer halves ----
constexpr int kTraceHalf = 512;  // events per CTA per role
enum : uint16_t { EV_WAIT0 = 1, EV_WAIT1, EV_ISSUED, EV_FIRST, EV_DONE, EV_PUB, EV_ENTRY, EV_EXIT,
                  EV_START, EV_LEFT, EV_X1, EV_X2, EV_X3 };

__device__ __forceinline__ void trace_ev(const AllreduceArgs& a, int role, int& n, uint16_t ev,
                                         int seg) {
  if (!a.trace || n >= kTraceHalf) return;
  TraceEv* e = a.trace + (static_cast<int64_t>(blockIdx.x) * 3 + role) * kTraceHalf + n++;
  e->t = globaltimer_ns();
  e->cta = blockIdx.x;
  e->ev = ev;
  e->seg = static_cast<uint16_t>(seg);
}

// Entry barrier + length agreement. Returns false if this view must skip work.
__device__ bool entry_barrier(const AllreduceArgs& a, const ViewArgs& v, int local_cta,
                              uint32_t epoch) {
  const int tid = threadIdx.x;
  const unsigned long long mylen =
      static_cast<unsigned long long>(a.n) | (static_cast<unsigned long long>(a.n_workers) << 56);
  if (local_cta == 0 && tid < a.n_ranks && tid != v.rank) {
    Ctrl* pc = v.peer_ctrl[tid];
    st_relaxed_sys64(reinterpret_cast<uint64_t*>(&pc->arrive_len[v.rank]), mylen);
    st_relaxed_sys64(reinterpret_cast<uint64_t*>(&pc->arrive_cfg[v.rank]), a.cfg_word);
    st_release_sys(&pc->arrive_epoch[v.rank], epoch);  // (release: orders both words first)
  }
  __shared__ int s_ok;
  if (tid == 0) {
    int ok = 1;
    for (int r = 0; r < a.n_ranks && ok; ++r) {
      if (r == v.rank) continue;
      if (!wait_flag(v, &v.ctrl->arrive_epoch[r], epoch, a.timeout_ns, 1000 + r)) {
        ok = 0;
        break;
      }
      unsigned long long len =
          ld_relaxed_sys64(reinterpret_cast<const uint64_t*>(&v.ctrl->arrive_len[r]));
      if (len != mylen) {
        // every rank sees the same table, so every rank reports the mismatch
        if (local_cta == 0) raise_err(v, MD_ERR_LENGTH_MISMATCH, r);
        ok = 0;
      } else if (ld_relaxed_sys64(reinterpret_cast<const uint64_t*>(&v.ctrl->arrive_cfg[r])) !=
                 a.cfg_word) {
        if (local_cta == 0) raise_err(v, MD_ERR_INVALID_CONFIG, 8000 + r);
        ok = 0;
      }
    }
    s_ok = ok;
  }
  __syncthreads();
  return s_ok != 0;
}

// The done flag only certifies "every read this rank made of your memory has
// completed": those reads were consumed (TMA completion / register use)
// before the CTA got here, and every datum a peer reads from us was already
// released by its segment flag. So (flag_gpu_fence) a GPU-scope acq_rel
// counter orders the CTAs and relaxed system-scope stores carry the flag --
// the two sys fences this replaces cost ~5 us per call (profiles/README.md).
__device__ void exit_barrier(const AllreduceArgs& a, const ViewArgs& v, uint32_t epoch) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t prev;
    if (a.flag_gpu_fence) {
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                   : "=r"(prev) : "l"(&v.ctrl->finished) : "memory");
    } else {
      __threadfence_system();
      prev = atomicAdd(&v.ctrl->finished, 1u);
    }
    s_last = (prev == static_cast<uint32_t>(a.ctas_per_view - 1));
  }
  __syncthreads();
  if (!s_last) return;
  // last CTA of this rank: nobody here reads peer memory any more
  const int tid = threadIdx.x;
  int tn = kTraceHalf - 8;  // (the channels kernel logs its own events in the last 4 slots)
  if (tid == 0) trace_ev(a, 0, tn, EV_X1, 0);
  if (tid < a.n_ranks && tid != v.rank) {
    if (a.flag_gpu_fence && !a.exit_sys_release) {
      st_relaxed_sys(&v.peer_ctrl[tid]->done_epoch[v.rank], epoch);
    } else {
      // owner-push: the flag also certifies our bulk stores INTO the peer
      // (complete per wait_group 0 in every CTA, ordered by the acq_rel CTA
      // counter); a system-scope release makes that formal, once per call
      if (!a.flag_gpu_fence) __threadfence_system();
      st_release_sys(&v.peer_ctrl[tid]->done_epoch[v.rank], epoch);
    }
  }
  __syncthreads();
  if (tid == 0) trace_ev(a, 0, tn, EV_X2, 0);
  if (tid == 0) {
    for (int r = 0; r < a.n_ranks; ++r) {
      if (r == v.rank) continue;
      // abort does not short-circuit here: peers still need our done flag,
      // and theirs bound the time anybody may still read our buffer
      uint64_t t0 = globaltimer_ns();
      while (!epoch_ge(ld_acquire_sys(&v.ctrl->done_epoch[r]), epoch)) {
        if (globaltimer_ns() - t0 > a.timeout_ns) {
          raise_err(v, MD_ERR_TIMEOUT, 2000 + r);
          break;
        }
        __nanosleep(32);
      }
    }
    trace_ev(a, 0, tn, EV_X3, 0);  // every peer's done flag seen
    v.ctrl->queue_head = 0;
    v.ctrl->finished = 0;
    v.ctrl->abort_flag = 0;
    v.ctrl->epoch = epoch;
    __threadfence();
  }
}

template <int kEpi>
__global__ void __launch_bounds__(kArThreads, 1)
    allreduce_kernel(const __grid_constant__ AllreduceArgs a) {
  const int view = blockIdx.x / a.ctas_per_view;
  const int local_cta = blockIdx.x % a.ctas_per_view;
  const ViewArgs& v = a.v[view];
  const RankPlan& rp = a.plan[v.rank];
  const int tid = threadIdx.x, nthr = blockDim.x;

  // the epoch lives in the control block (device side), so a captured CUDA
  // graph can replay this launch: every call bumps it exactly once
  __shared__ uint32_t s_epoch;
  __shared__ __align__(8) uint64_t tma_full[kStages];
  extern __shared__ __align__(128) char ring[];  // kRingBytes of TMA stages
  uint32_t tma_seq = 0;                          // chunks through the ring so far
  if (tid == 0) {
    s_epoch = *reinterpret_cast<volatile uint32_t*>(&v.ctrl->epoch) + 1;
    for (int s = 0; s < kStages; ++s) mbar_init(&tma_full[s], 1);
    mbar_init_fence();
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;
  bool ok = entry_barrier(a, v, local_cta, epoch);
  const int n_tasks = rp.n_tasks;
  // queue order: "time" tau, then task (tasks are sorted by stage); task t
  // works on segment tau - lag * stage(t), so a consumer is handed its
  // segment about `lag` segments after the producer stage was handed it --
  // late enough that its flag is usually already set. Producers always come
  // strictly earlier in this order, which keeps flag waits deadlock free.
  const int64_t n_items =
      static_cast<int64_t>(a.max_nseg + a.lag * a.max_stage) * n_tasks;
  __shared__ int64_t s_item;
  __shared__ int s_go;

  while (ok) {
    if (tid == 0) {
      s_item = atomicAdd(&v.ctrl->queue_head, 1u);
      if (*reinterpret_cast<volatile uint32_t*>(&v.ctrl->abort_flag)) s_item = n_items;
    }
    __syncthreads();
    const int64_t item = s_item;
    if (item >= n_items) break;
    const Task& t = rp.t[item % n_tasks];
    const int s = static_cast<int>(item / n_tasks) - a.lag * t.stage;
    int64_t cstart, clen;
    chunk_of(a.n, a.k, t.color, &cstart, &clen);
    if (s < 0 || s >= nseg_of(cstart, clen, a.seg)) {
      __syncthreads();
      continue;
    }
    // a non-root leaf without a worker fold has nothing to do: its data was
    // ready at the entry barrier (a lone root still runs its epilogue)
    if (t.type == 0 && t.is_leaf && t.parent >= 0 && a.n_workers == 0) {
      __syncthreads();
      continue;
    }
    const int64_t A = cstart & ~int64_t(3);
    const int64_t lo = max(cstart, A + static_cast<int64_t>(s) * a.seg);
    const int64_t hi = min(cstart + clen, A + static_cast<int64_t>(s + 1) * a.seg);

    // ---- wait for producers
    if (tid == 0) {
      int go = 1;
      if (t.type == 1) {
        go = wait_flag(v, &v.ctrl->down[t.color][s], epoch, a.timeout_ns, 3000 + t.color);
      } else {
        for (int j = 0; j < t.n_fold && go; ++j) {
          if (t.fold_src[j] == v.rank) continue;
          if (t.fold_leaf[j] && a.n_workers == 0) continue;
          go = wait_flag(v, &v.ctrl->up[t.color][j][s], epoch, a.timeout_ns, 4000 + t.color);
        }
      }
      s_go = go;
    }
    __syncthreads();
    if (!s_go) break;

    // ---- data
    const bool final_here = (t.type == 1) || (t.parent < 0);
    const int64_t vlo = min(hi, (lo + 3) & ~int64_t(3));
    const int64_t vhi = max(vlo, hi & ~int64_t(3));
    if (a.vec_ok) {
      const int nrem = t.type == 1 ? 1 : t.n_fold - 1;  // UP folds always hold the own value
      if (nrem >= 1 && vhi > vlo)
        item_tma<kEpi>(a, v, t, final_here, vlo, vhi, nrem, ring, tma_full, tma_seq);
      else
        item_dispatch<true, kEpi>(a, v, t, final_here, vlo, vhi, tid, nthr);
      if (tid < 8) {  // <= 3 head + <= 3 tail scalars
        int64_t i = (tid < 4) ? lo + tid : vhi + (tid - 4);
        bool mine = (tid < 4) ? (i < vlo) : (i < hi);
        if (mine) item_dispatch<false, kEpi>(a, v, t, final_here, i, i + 1, 0, 1);
      }
    } else {
      item_dispatch<false, kEpi>(a, v, t, final_here, lo, hi, tid, nthr);
    }
    __syncthreads();

    // ---- publish
    if (t.type == 0 && t.parent >= 0) {
      if (tid == 0) {
        __threadfence_system();
        st_release_sys(&v.peer_ctrl[t.parent]->up[t.color][t.my_slot][s], epoch);
      }
    } else if (final_here) {
      if (tid < t.n_down) {
        __threadfence_system();
        st_release_sys(&v.peer_ctrl[t.down[tid]]->down[t.color][s], epoch);
      }
    }
  }
  exit_barrier(a, v, epoch);
}

// ---- channelized kernel (vector-aligned buffers) -------------------------------
// Every CTA owns one task of its rank (UP fold or DOWN copy of one color) and
// the segments idx, idx + m, idx + 2m, ... of that task's chunk, where the m
// CTAs of a task are allotted in proportion to its remote bytes. Inside a CTA
// warp 0 is the producer: it waits for each segment's flags, handles the <= 3
// unaligned edge elements itself and streams the remote sources through the
// TMA ring; warps 1.. are consumers: fold (reference order), store, SGD
// epilogue, and publish the segment's flag. The ring runs continuously across
// the CTA's segments, so NVLink transfers, HBM epilogue and flag latency all
// overlap; segments can stay small (fine-grained pipelining across GPUs).
// warp 0: TMA producer, warp 1: notifier (publishes finished segments, so the
// flag fences never stall the consumers), warps 2..15: consumers
constexpr int kConsumerWarps = kArThreads / 32 - 2;
constexpr int kConsumerBase = 64;
constexpr int kDoneSlots = 8;  // segments a notifier may lag behind the consumers

__device__ __forceinline__ int task_weight(const AllreduceArgs& a, const Task& t) {
  if (t.type == 1) return 1;                                   // DOWN: one remote source
  if (t.n_fold > 1) return t.n_fold - 1;                       // UP with children
  return (t.parent < 0 || a.n_workers > 0) ? 1 : 0;            // lone root / leaf fold
}

// Deterministic CTA -> (task, index, count) allotment, identical in every CTA.
__device__ void allot(const AllreduceArgs& a, const RankPlan& rp, int cta, int* task, int* idx,
                      int* count) {
  int m[2 * MD_MAX_COLORS];
  int w[2 * MD_MAX_COLORS];
  int W = 0, used = 0;
  for (int i = 0; i < rp.n_tasks; ++i) {
    w[i] = task_weight(a, rp.t[i]);
    W += w[i];
  }
  *task = -1;
  if (W == 0) return;
  for (int i = 0; i < rp.n_tasks; ++i) {
    m[i] = w[i] ? max(1, a.ctas_per_view * w[i] / W) : 0;
    used += m[i];
  }
  while (used > a.ctas_per_view) {  // too many tasks for the CTAs: trim the largest
    int big = 0;
    for (int i = 1; i < rp.n_tasks; ++i)
      if (m[i] > m[big]) big = i;
    if (m[big] <= 1) break;
    --m[big];
    --used;
  }
  for (int i = 0; used < a.ctas_per_view; i = (i + 1) % rp.n_tasks)  // spread the rest
    if (w[i]) {
      ++m[i];
      ++used;
    }
  int base = 0;
  for (int i = 0; i < rp.n_tasks; ++i) {
    if (cta < base + m[i]) {
      *task = i;
      *idx = cta - base;
      *count = m[i];
      return;
    }
    base += m[i];
  }
}

struct SegGeom {
  int64_t lo, hi, vlo, vhi, C, nch;
};

__device__ __forceinline__ SegGeom seg_geom(const AllreduceArgs& a, const Task& t, int s,
                                            int nslot) {
  int64_t cstart, clen;
  chunk_of(a.n, a.k, t.color, &cstart, &clen);
  const int64_t A = cstart & ~int64_t(3);
  SegGeom g;
  g.lo = max(cstart, A + static_cast<int64_t>(s) * a.seg);
  g.hi = min(cstart + clen, A + static_cast<int64_t>(s + 1) * a.seg);
  g.vlo = min(g.hi, (g.lo + 3) & ~int64_t(3));
  g.vhi = max(g.vlo, g.hi & ~int64_t(3));
  g.C = nslot ? static_cast<int64_t>(kStageBytes / (4u * nslot)) & ~int64_t(3) : 0;
  g.nch = nslot ? (g.vhi - g.vlo + g.C - 1) / g.C : 0;
  return g;
}

// Wait (thread-level) for the producers of segment s of task t.
__device__ bool wait_inputs(const AllreduceArgs& a, const ViewArgs& v, const Task& t, int s,
                            uint32_t epoch) {
  if (t.type == 1) return wait_flag(v, &v.ctrl->down[t.color][s], epoch, a.timeout_ns, 3000 + t.color);
  for (int j = 0; j < t.n_fold; ++j) {
    if (t.fold_src[j] == v.rank) continue;
    if (t.fold_leaf[j] && a.n_workers == 0) continue;
    if (!wait_flag(v, &v.ctrl->up[t.color][j][s], epoch, a.timeout_ns, 4000 + t.color))
      return false;
  }
  return true;
}

// Release segment s: up flag in the parent, or down flags in the children.
// Flag stores of segment s; `fence` = issue the release fence first (the
// notifier batches several segments behind one fence).
// Default (sys fence): st.release.sys is cumulative -- it orders every store
// that precedes it in causality order (the consumers' stores via the
// mbarriers, the producer's edge stores) before the flag.
// flag_gpu_fence: one fence.acq_rel.gpu, then relaxed system-scope flag
// stores. Every flag certifies data in the PUBLISHER's own HBM, and peers
// read it through the publisher's L2; a GPU-scope fence already makes our
// stores visible there, without the sys fence's wait for the SM's in-flight
// NVLink traffic (measured 49 us vs 11 us per segment, profiles/README.md).
__device__ __forceinline__ void publish_flags(const AllreduceArgs& a, const ViewArgs& v,
                                              const Task& t, int s, uint32_t epoch, bool fence) {
  const bool up = t.type == 0 && t.parent >= 0;
  if (!up && t.n_down == 0) return;  // nobody waits for this segment
  if (fence && a.flag_gpu_fence) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  if (up) {
    uint32_t* f = &v.peer_ctrl[t.parent]->up[t.color][t.my_slot][s];
    if (a.flag_gpu_fence) st_relaxed_sys(f, epoch);
    else st_release_sys(f, epoch);
  } else {
    for (int c = 0; c < t.n_down; ++c) {
      uint32_t* f = &v.peer_ctrl[t.down[c]]->down[t.color][s];
      if (a.flag_gpu_fence) st_relaxed_sys(f, epoch);
      else st_release_sys(f, epoch);
    }
  }
}

__device__ __forceinline__ void publish(const AllreduceArgs& a, const ViewArgs& v, const Task& t,
                                        int s, uint32_t epoch) {
  publish_flags(a, v, t, s, epoch, true);
}

__device__ __forceinline__ bool aborted(const ViewArgs& v) {
  return *reinterpret_cast<volatile uint32_t*>(&v.ctrl->abort_flag) != 0;
}

template <int kEpi>
__device__ void run_channel(const AllreduceArgs& a, const ViewArgs& v, const Task& t, int idx,
                            int m, uint32_t epoch, char* ring, uint64_t* full, uint64_t* empty,
                            uint64_t* done, uint64_t* ack, const FoldProg& prog) {
  const int tid = threadIdx.x;
  const bool final_here = (t.type == 1) || (t.parent < 0);
  const int nrem = t.type == 1 ? 1 : t.n_fold - 1;
  int64_t cstart, clen;
  chunk_of(a.n, a.k, t.color, &cstart, &clen);
  const int nseg = static_cast<int>(nseg_of(cstart, clen, a.seg));

  // local-only tasks (lone root epilogue, leaf worker fold) stream with plain
  // 16-byte loads: for pure HBM traffic that measured faster than the TMA ring
  // (81 % vs 72 % of HBM at N = 1, profiles/README.md)
  if (nrem == 0) {
    for (int s0 = idx; s0 < nseg; s0 += m) {
      // last segments first: a producer that just streamed the buffer (the
      // step's gradient fill) left its END most recently in L2
      const int s = a.reverse_local ? nseg - 1 - s0 : s0;
      SegGeom g = seg_geom(a, t, s, 0);
      if (kEpi != 0 && final_here && t.type == 0 && t.n_fold == 1 && a.n_workers == 0)
        lone_update<kEpi>(a, v, g.vlo, g.vhi, tid, blockDim.x);
      else
        item_dispatch<true, kEpi>(a, v, t, final_here, g.vlo, g.vhi, tid, blockDim.x);
      if (tid < 8) {
        int64_t i = (tid < 4) ? g.lo + tid : g.vhi + (tid - 4);
        bool mine = (tid < 4) ? (i < g.vlo) : (i < g.hi);
        if (mine) item_dispatch<false, kEpi>(a, v, t, final_here, i, i + 1, 0, 1);
      }
      __syncthreads();
      if (tid == 0 && !(t.type == 0 && t.parent < 0 && t.n_down == 0)) publish(a, v, t, s, epoch);
    }
    return;
  }

  // Every input of a chunk arrives by TMA into one ring stage, laid out as
  // [remote sources in fold order][own value][W][momentum] (slots of C floats),
  // so the consumers never wait on a global load: they read SMEM and issue
  // fire-and-forget stores.
  const bool tma_own = t.type != 1 && a.n_workers == 0;  // worker folds stay LDG
  const bool owner = t.type == 2;  // stage slot r = rank r (own included), then W, momentum
  constexpr bool kMomT = kEpi >= 3;
  const bool tma_epi = kEpi != 0 && final_here;
  const int own_slot = nrem;
  const int w_slot = nrem + (tma_own ? 1 : 0);
  const int m_slot = w_slot + 1;
  const int nslot = w_slot + (tma_epi ? (kMomT ? 2 : 1) : 0);
  const int64_t ulen4 = a.update_len & ~int64_t(3);  // W/momentum rows TMA may read

  if (tid < 32) {  // ---------------- producer warp (lane 0 works) ----------------
    if (tid != 0) return;
    uint32_t gseq = 0;
    int pn = 0;  // trace events
    for (int s = idx; s < nseg; s += m) {
      SegGeom g = seg_geom(a, t, s, nslot);
      trace_ev(a, 0, pn, EV_WAIT0, s);
      if (!wait_inputs(a, v, t, s, epoch)) return;
      trace_ev(a, 0, pn, EV_WAIT1, s);
      fence_proxy_async_global();
      // unaligned edges (only the first/last segment of a color has any)
      for (int64_t i = g.lo; i < g.hi; ++i) {
        if (i >= g.vlo && i < g.vhi) {
          i = g.vhi - 1;
          continue;
        }
        item_dispatch<false, kEpi>(a, v, t, final_here, i, i + 1, 0, 1);
      }
      if (g.nch == 0) {  // nothing for the consumers: release the segment here
        publish(a, v, t, s, epoch);
        continue;
      }
      for (int64_t c = 0; c < g.nch; ++c, ++gseq) {
        const uint32_t st = gseq % kStages;
        if (gseq >= kStages) {
          uint32_t spins = 0;
          while (!mbar_try_wait(&empty[st], ((gseq / kStages) - 1) & 1)) {
            if ((++spins & 1023) == 0 && aborted(v)) return;
          }
        }
        const int64_t clo = g.vlo + c * g.C;
        const int64_t chi = min(g.vhi, clo + g.C);
        const uint32_t bytes = static_cast<uint32_t>((chi - clo) * 4);
        uint32_t wbytes = 0;
        if (tma_epi) {
          const int64_t whi = min(chi, ulen4);
          wbytes = whi > clo ? static_cast<uint32_t>((whi - clo) * 4) : 0u;
        }
        char* stage = ring + st * kStageBytes;
        const size_t slot = static_cast<size_t>(g.C) * 4;
        mbar_expect_tx(&full[st], bytes * (nrem + (tma_own ? 1 : 0)) + wbytes * (kMomT ? 2 : 1));
        if (t.type == 1) {
          tma_load_1d(stage, v.peer[t.parent] + clo, bytes, &full[st]);
        } else if (owner) {
          for (int r = 0; r < a.n_ranks; ++r)
            tma_load_1d(stage + r * slot, (r == v.rank ? v.buf : v.peer[r]) + clo, bytes, &full[st]);
        } else {
          int q = 0;
          for (int j = 0; j < t.n_fold; ++j) {
            const int src = t.fold_src[j];
            if (src == v.rank) continue;
            tma_load_1d(stage + q * slot, v.peer[src] + clo, bytes, &full[st]);
            ++q;
          }
          if (tma_own) tma_load_1d(stage + own_slot * slot, v.buf + clo, bytes, &full[st]);
        }
        if (wbytes) {
          tma_load_1d(stage + w_slot * slot, v.w + clo, wbytes, &full[st]);
          if (kMomT) tma_load_1d(stage + m_slot * slot, v.mom + clo, wbytes, &full[st]);
        }
      }
      trace_ev(a, 0, pn, EV_ISSUED, s);
    }
    return;
  }

  if (tid < kConsumerBase) {  // ---------------- notifier warp (lane 0) ----------------
    if (tid != 32) return;
    int cn = 0;  // trace events
    uint32_t j = 0;  // consumer-visible segments seen
    int pend[kDoneSlots];
    int npend = 0;
    for (int s = idx; s < nseg; s += m) {
      SegGeom g = seg_geom(a, t, s, nslot);
      if (g.nch == 0) continue;
      pend[npend++] = s;
      uint32_t spins = 0;
      while (!mbar_try_wait(&done[j % kDoneSlots], (j / kDoneSlots) & 1)) {
        if ((++spins & 1023) == 0 && aborted(v)) return;
      }
      ++j;
      // batch: also take every following segment that is already finished
      int s2 = s + m;
      while (npend < kDoneSlots && s2 < nseg) {
        SegGeom g2 = seg_geom(a, t, s2, nslot);
        if (g2.nch == 0) {
          s2 += m;
          continue;
        }
        if (!mbar_try_wait(&done[j % kDoneSlots], (j / kDoneSlots) & 1)) break;
        pend[npend++] = s2;
        ++j;
        s = s2;
        s2 += m;
      }
      trace_ev(a, 2, cn, EV_DONE, pend[npend - 1]);
      for (int i = 0; i < npend; ++i) publish_flags(a, v, t, pend[i], epoch, i == 0);
      trace_ev(a, 2, cn, EV_PUB, pend[npend - 1]);
      for (int i = 0; i < npend; ++i) {  // free the done slots for the consumers
        const uint32_t jj = j - npend + i;
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&ack[jj % kDoneSlots]))
                     : "memory");
      }
      npend = 0;
    }
    return;
  }

  // ---------------- consumer warps ----------------
  const int ct = tid - kConsumerBase, nct = kConsumerWarps * 32;
  uint32_t gseq = 0, jseg = 0;
  int cn = 0;  // trace events (ct == 0 only)
  for (int s = idx; s < nseg; s += m) {
    SegGeom g = seg_geom(a, t, s, nslot);
    if (g.nch == 0) continue;
    const size_t slot4 = static_cast<size_t>(g.C) / 4;  // float4 per slot
    for (int64_t c = 0; c < g.nch; ++c, ++gseq) {
      const uint32_t st = gseq % kStages;
      uint32_t spins = 0;
      while (!mbar_try_wait(&full[st], (gseq / kStages) & 1)) {
        if ((++spins & 1023) == 0 && aborted(v)) return;
      }
      if (c == 0 && ct == 0) trace_ev(a, 1, cn, EV_FIRST, s);
      const float4* stage = reinterpret_cast<const float4*>(ring + st * kStageBytes);
      const int64_t clo = g.vlo + c * g.C;
      const int64_t chi = min(g.vhi, clo + g.C);
      const int64_t n4 = (chi - clo) / 4;
#pragma unroll 2
      for (int64_t e = ct; e < n4; e += nct) {
        const int64_t i = clo + 4 * e;
        float4 acc;
        if (t.type == 1) {
          acc = stage[e];
        } else if (owner) {  // the element's own color program over the rank slots
          float* sf = reinterpret_cast<float*>(ring + st * kStageBytes);
          const int c0 = color_of(a.n, a.prog_k, i);
          if (color_of(a.n, a.prog_k, i + 3) == c0) {
            acc = fold_prog4(prog.c[c0], sf, g.C, 4 * e);
          } else {
            acc.x = fold_prog(prog.c[c0], sf, g.C, 4 * e);
            acc.y = fold_prog(prog.c[color_of(a.n, a.prog_k, i + 1)], sf, g.C, 4 * e + 1);
            acc.z = fold_prog(prog.c[color_of(a.n, a.prog_k, i + 2)], sf, g.C, 4 * e + 2);
            acc.w = fold_prog(prog.c[color_of(a.n, a.prog_k, i + 3)], sf, g.C, 4 * e + 3);
          }
        } else {
          int q = 0;
          for (int jf = 0; jf < t.n_fold; ++jf) {
            float4 x;
            if (t.fold_src[jf] == v.rank) {
              x = tma_own ? stage[own_slot * slot4 + e] : own_value<true>(a, v, i);
            } else {
              x = stage[q * slot4 + e];
              ++q;
            }
            acc = (jf == 0) ? x : add4(acc, x);
          }
        }
        *reinterpret_cast<float4*>(v.buf + i) = acc;
        if constexpr (kEpi != 0) {
          if (final_here) {
            if (i + 4 <= ulen4) {  // W / momentum rows arrived with the chunk
              float4 w = stage[w_slot * slot4 + e];
              float4 mm = kMomT ? stage[m_slot * slot4 + e] : make_float4(0.f, 0.f, 0.f, 0.f);
              sgd_elem<kEpi>(w.x, acc.x, mm.x, a);
              sgd_elem<kEpi>(w.y, acc.y, mm.y, a);
              sgd_elem<kEpi>(w.z, acc.z, mm.z, a);
              sgd_elem<kEpi>(w.w, acc.w, mm.w, a);
              __stcs(reinterpret_cast<float4*>(v.w + i), w);
              if (kMomT) __stcs(reinterpret_cast<float4*>(v.mom + i), mm);
            } else {  // the ragged tail of the update range
              epi_scalar<kEpi>(a, v, i, acc.x);
              epi_scalar<kEpi>(a, v, i + 1, acc.y);
              epi_scalar<kEpi>(a, v, i + 2, acc.z);
              epi_scalar<kEpi>(a, v, i + 3, acc.w);
            }
          }
        }
      }
      __syncwarp();
      if ((ct & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&empty[st])) : "memory");
    }
    // this warp is done with segment s: tell the notifier (the slot must have
    // been acknowledged for the segment kDoneSlots earlier)
    if ((ct & 31) == 0) {
      if (jseg >= kDoneSlots) {
        uint32_t spins = 0;
        while (!mbar_try_wait(&ack[jseg % kDoneSlots], ((jseg / kDoneSlots) - 1) & 1)) {
          if ((++spins & 1023) == 0 && aborted(v)) return;
        }
      }
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&done[jseg % kDoneSlots]))
                   : "memory");
    }
    __syncwarp();
    ++jseg;
  }
}

template <int kEpi>
__global__ void __launch_bounds__(kArThreads, 1)
    allreduce_channels_kernel(const __grid_constant__ AllreduceArgs a) {
  const int view = blockIdx.x / a.ctas_per_view;
  const int local_cta = blockIdx.x % a.ctas_per_view;
  const ViewArgs& v = a.v[view];
  const RankPlan& rp = a.plan[v.rank];
  const int tid = threadIdx.x;
  __shared__ uint32_t s_epoch;
  __shared__ __align__(8) uint64_t full[kStages];
  __shared__ __align__(8) uint64_t empty[kStages];
  __shared__ __align__(8) uint64_t done[kDoneSlots];
  __shared__ __align__(8) uint64_t ack[kDoneSlots];
  __shared__ int s_task, s_idx, s_m;
  __shared__ FoldProg prog;  // owner schedule only
  extern __shared__ __align__(128) char ring[];
  if (a.prog)
    for (int i = tid; i < static_cast<int>(sizeof(FoldProg) / 4); i += blockDim.x)
      reinterpret_cast<uint32_t*>(&prog)[i] = reinterpret_cast<const uint32_t*>(a.prog)[i];
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    for (int s = 0; s < kDoneSlots; ++s) {
      mbar_init(&done[s], kConsumerWarps);
      mbar_init(&ack[s], 1);
    }
    mbar_init_fence();
    int task, idx = 0, m = 1;
    allot(a, rp, local_cta, &task, &idx, &m);
    s_task = task;
    s_idx = idx;
    s_m = m;
  }
  if (tid == 0) s_epoch = *reinterpret_cast<volatile uint32_t*>(&v.ctrl->epoch) + 1;
  __syncthreads();
  const uint32_t epoch = s_epoch;
  int tn = kTraceHalf - 4;  // kernel-level events in the producer half's last slots
  if (tid == 0) trace_ev(a, 0, tn, EV_START, s_task < 0 ? 0xffff : s_task);
  const bool ok = entry_barrier(a, v, local_cta, epoch);
  if (tid == 0) trace_ev(a, 0, tn, EV_ENTRY, s_task < 0 ? 0xffff : s_task);
  if (ok && s_task >= 0)
    run_channel<kEpi>(a, v, rp.t[s_task], s_idx, s_m, epoch, ring, full, empty, done, ack, prog);
  __syncthreads();
  if (tid == 0) trace_ev(a, 0, tn, EV_EXIT, s_task < 0 ? 0xffff : s_task);
  exit_barrier(a, v, epoch);
  if (tid == 0) trace_ev(a, 0, tn, EV_LEFT, s_task < 0 ? 0xffff : s_task);
}

// ---- one-shot kernel (latency path: small and mid-size buffers) ---------------
// Every rank pulls the WHOLE buffer of every peer (one NVLink round trip per
// CTA, all sources in flight at once through TMA) and evaluates every color's
// fold locally with the color's fold program -- the same adds in the same
// order as the tree schedule, so the same bits (ColorProg). No per-segment
// flags, no UP -> DOWN dependency chain: entry barrier, one read, a
// "read done" barrier (the exit barrier's done flags, moved before the
// in-place writes: nobody overwrites a buffer a peer still reads), fold +
// SGD epilogue + store. Ingress is (N-1) x bytes instead of the tree's
// 2 (N-1)/N x bytes: equal at N = 2, so there it serves every size that fits
// one SMEM pass (N x E floats per CTA <= kRingBytes); at larger N only small
// and mid-size buffers (host threshold, md_allreduce).
// all CTAs of this rank: count in; the last tells every peer "I have finished
// reading your buffer" (done flag); then every CTA waits for every peer's.
__device__ void read_done_barrier(const AllreduceArgs& a, const ViewArgs& v, uint32_t epoch,
                                  int ctas) {
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(prev) : "l"(&v.ctrl->finished) : "memory");
    if (prev == static_cast<uint32_t>(ctas - 1)) {
      for (int r = 0; r < a.n_ranks; ++r)
        if (r != v.rank) st_relaxed_sys(&v.peer_ctrl[r]->done_epoch[v.rank], epoch);
    }
    for (int r = 0; r < a.n_ranks; ++r) {
      if (r == v.rank) continue;
      uint64_t t0 = globaltimer_ns();
      while (!epoch_ge(ld_acquire_sys(&v.ctrl->done_epoch[r]), epoch)) {
        if (globaltimer_ns() - t0 > a.timeout_ns) {
          raise_err(v, MD_ERR_TIMEOUT, 2000 + r);
          break;
        }
        __nanosleep(20);
      }
    }
  }
  __syncthreads();
}

// Fold every color's program over the staged rank slots [N][E] for elements
// [lo, hi), store the sums in place and apply the fused SGD epilogue.
template <int kEpi>
__device__ void fold_store_range(const AllreduceArgs& a, const ViewArgs& v, const FoldProg& prog,
                                 float* slots, int64_t E, int64_t lo, int64_t hi) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int64_t len = hi - lo;
  for (int64_t e = 4 * tid; e < len; e += 4 * nthr) {
    const int64_t i = lo + e;
    const int c0 = color_of(a.n, a.k, i);
    if (e + 4 <= len && color_of(a.n, a.k, i + 3) == c0) {
      const float4 g = fold_prog4(prog.c[c0], slots, E, e);
      *reinterpret_cast<float4*>(v.buf + i) = g;
      if constexpr (kEpi != 0) {
        if (i + 4 <= a.update_len) {
          constexpr bool kMom = kEpi >= 3;
          float4 w = *reinterpret_cast<const float4*>(v.w + i);
          float4 m = kMom ? *reinterpret_cast<const float4*>(v.mom + i)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
          sgd_elem<kEpi>(w.x, g.x, m.x, a);
          sgd_elem<kEpi>(w.y, g.y, m.y, a);
          sgd_elem<kEpi>(w.z, g.z, m.z, a);
          sgd_elem<kEpi>(w.w, g.w, m.w, a);
          *reinterpret_cast<float4*>(v.w + i) = w;
          if (kMom) *reinterpret_cast<float4*>(v.mom + i) = m;
        } else {
          epi_scalar<kEpi>(a, v, i, g.x);
          epi_scalar<kEpi>(a, v, i + 1, g.y);
          epi_scalar<kEpi>(a, v, i + 2, g.z);
          epi_scalar<kEpi>(a, v, i + 3, g.w);
        }
      }
    } else {
      for (int64_t q = e; q < min(len, e + 4); ++q) {
        const float g = fold_prog(prog.c[color_of(a.n, a.k, lo + q)], slots, E, q);
        v.buf[lo + q] = g;
        epi_scalar<kEpi>(a, v, lo + q, g);
      }
    }
  }
}

template <int kEpi>
__global__ void __launch_bounds__(kArThreads, 1)
    allreduce_oneshot_kernel(const __grid_constant__ AllreduceArgs a) {
  const int view = blockIdx.x / a.ctas_per_view;
  const int local_cta = blockIdx.x % a.ctas_per_view;
  const ViewArgs& v = a.v[view];
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int N = a.n_ranks;
  const int64_t E = a.seg;  // elements per CTA (multiple of 4)
  const int64_t lo = static_cast<int64_t>(local_cta) * E;
  const int64_t hi = min(a.n, lo + E);
  const int64_t vhi = max(lo, hi & ~int64_t(3));
  __shared__ uint32_t s_epoch;
  __shared__ __align__(8) uint64_t bar;
  __shared__ FoldProg prog;
  extern __shared__ __align__(128) char ring[];
  float* slots = reinterpret_cast<float*>(ring);  // [N][E]
  for (int i = tid; i < static_cast<int>(sizeof(FoldProg) / 4); i += nthr)
    reinterpret_cast<uint32_t*>(&prog)[i] = reinterpret_cast<const uint32_t*>(a.prog)[i];
  if (tid == 0) {
    s_epoch = *reinterpret_cast<volatile uint32_t*>(&v.ctrl->epoch) + 1;
    mbar_init(&bar, 1);
    mbar_init_fence();
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;
  const bool ok = entry_barrier(a, v, local_cta, epoch) && lo < hi;
  if (ok) {  // every rank's [lo, hi) into SMEM: N TMA copies in flight at once
    if (tid == 0 && vhi > lo) {
      fence_proxy_async_global();
      const uint32_t bytes = static_cast<uint32_t>((vhi - lo) * 4);
      mbar_expect_tx(&bar, bytes * N);
      for (int r = 0; r < N; ++r) tma_load_1d(slots + r * E, v.peer[r] + lo, bytes, &bar);
    }
    if (tid < 4 * N) {  // the <= 3 trailing elements of the buffer
      const int r = tid / 4;
      const int64_t i = vhi + (tid % 4);
      if (i < hi) slots[r * E + (i - lo)] = *reinterpret_cast<const volatile float*>(v.peer[r] + i);
    }
    if (vhi > lo)
      while (!mbar_try_wait(&bar, 0)) {
      }
  }
  read_done_barrier(a, v, epoch, a.ctas_per_view);
  if (ok && !aborted(v)) fold_store_range<kEpi>(a, v, prog, slots, E, lo, hi);
  // completion: the last CTA of the rank resets the per-call state (its own
  // counter: a CTA can get here while a sibling has not yet counted itself in
  // the read phase -- peers' done flags do not wait for our own reads)
  __syncthreads();
  if (tid == 0) {
    uint32_t prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(prev) : "l"(&v.ctrl->finished2) : "memory");
    if (prev == static_cast<uint32_t>(a.ctas_per_view - 1)) {
      v.ctrl->queue_head = 0;
      v.ctrl->finished = 0;
      v.ctrl->finished2 = 0;
      v.ctrl->abort_flag = 0;
      v.ctrl->epoch = epoch;
      __threadfence();
    }
  }
}

// ---- LL kernel (latency path: the smallest buffers) -----------------------------
// Push instead of pull: every rank stores its own values, each packed with the
// call's epoch into one 8-byte word, straight into every peer's LL inbox (a
// region of the peer-mapped control block), then polls its OWN inbox until
// every word carries the epoch. One NVLink one-way trip, no barrier, no flag
// fence: the epoch tag validates each word. The user buffers are never read
// remotely, so the result is stored in place at once (no read-done barrier),
// and the inbox parity (epoch & 1) cannot be overwritten before it was read:
// a sender is two calls ahead only after this rank pushed the call in between.
// The fold is the same fold program as the one-shot kernel -- same bits.
__device__ __forceinline__ void st_relaxed_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

template <int kEpi>
__global__ void __launch_bounds__(kArThreads, 1)
    allreduce_ll_kernel(const __grid_constant__ AllreduceArgs a) {
  const int view = blockIdx.x / a.ctas_per_view;
  const int local_cta = blockIdx.x % a.ctas_per_view;
  const ViewArgs& v = a.v[view];
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int N = a.n_ranks, me = v.rank;
  const int64_t E = a.seg;  // elements per CTA (multiple of 4)
  const int64_t lo = static_cast<int64_t>(local_cta) * E;
  const int64_t hi = min(a.n, lo + E);
  __shared__ uint32_t s_epoch;
  __shared__ int s_ok;
  __shared__ FoldProg prog;
  extern __shared__ __align__(128) char ring[];
  float* slots = reinterpret_cast<float*>(ring);  // [N][E]
  for (int i = tid; i < static_cast<int>(sizeof(FoldProg) / 4); i += nthr)
    reinterpret_cast<uint32_t*>(&prog)[i] = reinterpret_cast<const uint32_t*>(a.prog)[i];
  if (tid == 0) {
    s_epoch = *reinterpret_cast<volatile uint32_t*>(&v.ctrl->epoch) + 1;
    s_ok = 1;
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;
  const int par = epoch & 1;
  const unsigned long long tag = static_cast<unsigned long long>(epoch) << 32;
  // push my values to every peer's inbox (and stage them for my own fold)
  for (int64_t i = lo + tid; i < hi; i += nthr) {
    const float x = v.buf[i];
    slots[me * E + (i - lo)] = x;
    const unsigned long long word = tag | __float_as_uint(x);
    for (int r = 0; r < N; ++r)
      if (r != me) st_relaxed_sys_u64(&v.peer_ctrl[r]->ll[par][me][i], word);
  }
  // receive: every peer's word for every element of my range
  const uint64_t t0 = globaltimer_ns();
  for (int r = 0; r < N; ++r) {
    if (r == me) continue;
    const unsigned long long* box = v.ctrl->ll[par][r];
    for (int64_t i = lo + tid; i < hi; i += nthr) {
      unsigned long long w = ld_relaxed_sys_u64(box + i);
      uint32_t spins = 0;
      while (static_cast<uint32_t>(w >> 32) != epoch) {
        if ((++spins & 1023) == 0) {
          if (!s_ok || aborted(v)) break;
          if (globaltimer_ns() - t0 > a.timeout_ns) {
            raise_err(v, MD_ERR_TIMEOUT, 5000 + r);
            s_ok = 0;
            break;
          }
        }
        w = ld_relaxed_sys_u64(box + i);
      }
      slots[r * E + (i - lo)] = __uint_as_float(static_cast<uint32_t>(w));
    }
  }
  __syncthreads();
  if (s_ok && !aborted(v)) fold_store_range<kEpi>(a, v, prog, slots, E, lo, hi);
  __syncthreads();
  if (tid == 0) {
    uint32_t prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(prev) : "l"(&v.ctrl->finished2) : "memory");
    if (prev == static_cast<uint32_t>(a.ctas_per_view - 1)) {
      v.ctrl->finished2 = 0;
      v.ctrl->abort_flag = 0;
      v.ctrl->epoch = epoch;
      __threadfence();
    }
  }
}

// ---- stream kernel (all-pull, tiled; opt-in) --------------------------------------
// Every rank pulls every peer's buffer tile by tile through a TMA ring and
// folds each tile locally with the color fold programs (same bits as the
// tree schedule). At N = 2 the ingress equals the tree's (the whole peer
// buffer), but there is no UP -> DOWN dependency chain: no rank waits for
// another rank's fold, only for its READ of the tile about to be overwritten.
// Per tile: warp 0 issues the TMA loads (every rank's tile, plus the W and
// momentum rows of the epilogue); warp 1, once they landed, tells every peer
// "I have read your tile t" (rd flag in the peer's control block) and waits
// for the peers' flags for OUR tile t; warps 2.. fold the tile from SMEM, wait
// for that clearance, then store the sums in place and run the SGD epilogue.
// Peers read each tile at about the same time, so the clearance normally
// arrives while the fold runs. No exit barrier: every peer read of our buffer
// completed before the tile it read was overwritten.
// warp 0: TMA producer, warp 1: publisher, warp 2: clearance, warps 3..15: fold
constexpr int kStreamConsumerBase = 96;
constexpr int kStreamConsumerWarps = kArThreads / 32 - 3;

template <int kEpi>
__global__ void __launch_bounds__(kArThreads, 1)
    allreduce_stream_kernel(const __grid_constant__ AllreduceArgs a) {
  const int view = blockIdx.x / a.ctas_per_view;
  const int local_cta = blockIdx.x % a.ctas_per_view;
  const int G = a.ctas_per_view;
  const ViewArgs& v = a.v[view];
  const int tid = threadIdx.x;
  const int N = a.n_ranks, me = v.rank;
  const int64_t TE = a.seg;  // tile elements (multiple of 4)
  const int S = a.lag;       // ring stages
  const int64_t T = (a.n + TE - 1) / TE;
  constexpr bool kMom = kEpi >= 3;
  const size_t slot_f = static_cast<size_t>(TE);          // floats per slot
  const size_t stage_f = slot_f * (N + (kEpi == 0 ? 0 : (kMom ? 2 : 1)));  // [N ranks][W][mom]
  const int64_t ulen4 = a.update_len & ~int64_t(3);
  __shared__ uint32_t s_epoch;
  __shared__ __align__(8) uint64_t full[8], empty[8], clear[8];
  __shared__ FoldProg prog;
  extern __shared__ __align__(128) char ring[];
  float* ringf = reinterpret_cast<float*>(ring);
  for (int i = tid; i < static_cast<int>(sizeof(FoldProg) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(&prog)[i] = reinterpret_cast<const uint32_t*>(a.prog)[i];
  if (tid == 0) {
    s_epoch = *reinterpret_cast<volatile uint32_t*>(&v.ctrl->epoch) + 1;
    for (int st = 0; st < S; ++st) {
      mbar_init(&full[st], 1);
      // the publisher counts in too: a stage is refilled only after its
      // tile's read-done flags went out, so full[st] can never run a phase
      // ahead of the publisher (parity aliasing -> cross-GPU deadlock)
      mbar_init(&empty[st], kStreamConsumerWarps + 1);
      mbar_init(&clear[st], 1);
    }
    mbar_init_fence();
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;
  const bool ok = entry_barrier(a, v, local_cta, epoch);
  // the roles run in a lambda: an abort returns to the completion code below
  if (ok) [&]() {
    if (tid < 32) {  // ---------------- producer ----------------
      if (tid == 0) {
        fence_proxy_async_global();
        uint32_t seq = 0;
        for (int64_t t = local_cta; t < T; t += G, ++seq) {
          const uint32_t st = seq % S;
          if (seq >= static_cast<uint32_t>(S)) {
            uint32_t spins = 0;
            while (!mbar_try_wait(&empty[st], ((seq / S) - 1) & 1))
              if ((++spins & 1023) == 0 && aborted(v)) return;
          }
          const int64_t lo = t * TE, hi = min(a.n, lo + TE), vhi = max(lo, hi & ~int64_t(3));
          float* stage = ringf + st * stage_f;
          for (int64_t i = vhi; i < hi; ++i)  // <= 3 trailing elements of the buffer
            for (int r = 0; r < N; ++r)
              stage[r * slot_f + (i - lo)] = *reinterpret_cast<const volatile float*>(v.peer[r] + i);
          const uint32_t bytes = static_cast<uint32_t>((vhi - lo) * 4);
          uint32_t wbytes = 0;
          if (kEpi != 0) {
            const int64_t whi = min(vhi, ulen4);
            wbytes = whi > lo ? static_cast<uint32_t>((whi - lo) * 4) : 0u;
          }
          mbar_expect_tx(&full[st], bytes * N + wbytes * (kMom ? 2 : 1));
          if (bytes)
            for (int r = 0; r < N; ++r) tma_load_1d(stage + r * slot_f, v.peer[r] + lo, bytes, &full[st]);
          if (wbytes) {
            tma_load_1d(stage + N * slot_f, v.w + lo, wbytes, &full[st]);
            if (kMom) tma_load_1d(stage + (N + 1) * slot_f, v.mom + lo, wbytes, &full[st]);
          }
        }
      }
    } else if (tid < 64) {  // ---------------- publisher ----------------
      // "I have read your tile t" as soon as the tile landed -- never behind a
      // wait for the peers (that made every tile a cross-GPU round trip)
      if (tid == 32) {
        uint32_t seq = 0;
        for (int64_t t = local_cta; t < T; t += G, ++seq) {
          const uint32_t st = seq % S;
          uint32_t spins = 0;
          while (!mbar_try_wait(&full[st], (seq / S) & 1))
            if ((++spins & 1023) == 0 && aborted(v)) return;
          for (int r = 0; r < N; ++r)  // our reads of tile t completed (landed in SMEM)
            if (r != me) st_relaxed_sys(&v.peer_ctrl[r]->rd[me][t], epoch);
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&empty[st])) : "memory");
        }
      }
    } else if (tid < kStreamConsumerBase) {  // ---------------- clearance ----------------
      if (tid == 64) {
        uint32_t seq = 0;
        for (int64_t t = local_cta; t < T; t += G, ++seq) {
          const uint32_t st = seq % S;
          uint32_t spins = 0;
          // the stage holds tile t (so clear[st]'s previous phase was consumed)
          while (!mbar_try_wait(&full[st], (seq / S) & 1))
            if ((++spins & 1023) == 0 && aborted(v)) return;
          // relaxed polling: the flag orders nothing we read -- it only says the
          // peer's copy of our tile has landed, so our overwrite cannot reach it
          for (int r = 0; r < N; ++r) {
            if (r == me) continue;
            const uint32_t* f = &v.ctrl->rd[r][t];
            if (!epoch_ge(ld_relaxed_sys(f), epoch)) {
              const uint64_t t0 = globaltimer_ns();
              uint32_t sp = 0;
              while (!epoch_ge(ld_relaxed_sys(f), epoch)) {
                if ((++sp & 1023) == 0) {
                  if (aborted(v)) return;
                  if (globaltimer_ns() - t0 > a.timeout_ns) {
                    raise_err(v, MD_ERR_TIMEOUT, 6000 + r);
                    return;
                  }
                }
              }
            }
          }
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&clear[st])) : "memory");
        }
      }
    } else {  // ---------------- consumers ----------------
      const int ct = tid - kStreamConsumerBase, nct = kStreamConsumerWarps * 32;
      uint32_t seq = 0;
      for (int64_t t = local_cta; t < T; t += G, ++seq) {
        const uint32_t st = seq % S;
        const uint32_t par = (seq / S) & 1;
        uint32_t spins = 0;
        while (!mbar_try_wait(&full[st], par))
          if ((++spins & 1023) == 0 && aborted(v)) return;
        float* stage = ringf + st * stage_f;
        const int64_t lo = t * TE, len = min(a.n, lo + TE) - lo;
        // fold every element of the tile (results stay in SMEM: slot `root`)
        for (int64_t e = 4 * ct; e < len; e += 4 * nct) {
          const int c0 = color_of(a.n, a.k, lo + e);
          if (e + 4 <= len && color_of(a.n, a.k, lo + e + 3) == c0) {
            fold_prog4(prog.c[c0], stage, slot_f, e);
          } else {
            for (int64_t q = e; q < min(len, e + 4); ++q)
              fold_prog(prog.c[color_of(a.n, a.k, lo + q)], stage, slot_f, q);
          }
        }
        spins = 0;
        while (!mbar_try_wait(&clear[st], par))
          if ((++spins & 1023) == 0 && aborted(v)) return;
        for (int64_t e = 4 * ct; e < len; e += 4 * nct) {
          const int64_t i = lo + e;
          const int c0 = color_of(a.n, a.k, i);
          if (e + 4 <= len && color_of(a.n, a.k, i + 3) == c0) {
            const float4 g = *reinterpret_cast<const float4*>(stage + prog.c[c0].root * slot_f + e);
            __stcs(reinterpret_cast<float4*>(v.buf + i), g);
            if constexpr (kEpi != 0) {
              if (i + 4 <= ulen4) {
                float4 w = *reinterpret_cast<const float4*>(stage + N * slot_f + e);
                float4 m = kMom ? *reinterpret_cast<const float4*>(stage + (N + 1) * slot_f + e)
                                : make_float4(0.f, 0.f, 0.f, 0.f);
                sgd_elem<kEpi>(w.x, g.x, m.x, a);
                sgd_elem<kEpi>(w.y, g.y, m.y, a);
                sgd_elem<kEpi>(w.z, g.z, m.z, a);
                sgd_elem<kEpi>(w.w, g.w, m.w, a);
                __stcs(reinterpret_cast<float4*>(v.w + i), w);
                if (kMom) __stcs(reinterpret_cast<float4*>(v.mom + i), m);
              } else {
                epi_scalar<kEpi>(a, v, i, g.x);
                epi_scalar<kEpi>(a, v, i + 1, g.y);
                epi_scalar<kEpi>(a, v, i + 2, g.z);
                epi_scalar<kEpi>(a, v, i + 3, g.w);
              }
            }
          } else {
            for (int64_t q = e; q < min(len, e + 4); ++q) {
              const float g = stage[prog.c[color_of(a.n, a.k, lo + q)].root * slot_f + q];
              v.buf[lo + q] = g;
              epi_scalar<kEpi>(a, v, lo + q, g);
            }
          }
        }
        __syncwarp();
        if ((ct & 31) == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&empty[st])) : "memory");
      }
    }
  }();
  __syncthreads();
  if (tid == 0) {
    uint32_t prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(prev) : "l"(&v.ctrl->finished2) : "memory");
    if (prev == static_cast<uint32_t>(G - 1)) {
      v.ctrl->finished2 = 0;
      v.ctrl->finished = 0;
      v.ctrl->queue_head = 0;
      v.ctrl->abort_flag = 0;
      v.ctrl->epoch = epoch;
      __threadfence();
    }
  }
}

// ---- owner-push kernel (large buffers) ------------------------------------------
// Owner-computes with a PUSHED broadcast: rank j pulls slice j of every rank
// through a TMA ring, folds each element with its color program (same bits),
// and TMA-bulk-stores the final tile into its own buffer AND every peer's --
// no DOWN tasks, no per-segment flags. Slices are 16-byte aligned (the <= 3
// trailing elements of the buffer go to the last owner, scalar). A peer needs
// the pushes only at the end of the call, which the exit barrier's done flag
// certifies (each CTA waited for its bulk stores to complete). Pulls and
// pushes split the 2 (N-1)/N bytes per rank between the two directions of
// the links (measured ceilings ~650 / ~688 GB/s, profiles/README.md).
//
// Sharded SGD update (kEpi != 0; the host launches it only for
// MD_UPDATE_SHARDED): replicas are bitwise equal (ref sgd.py:5-10), so the
// owner of a slice may update it for everyone. The W and momentum rows of
// the owner's slice arrive with the tile, the fold warps apply the update in
// SMEM, and the storer pushes W' -- not g -- into every rank's weights, keeps
// the momentum rows local (sharded optimizer state) and stores g into its own
// buffer only. Buffer elements at or past update_len are pushed as in a
// plain call. Same NVLink bytes as the plain call, 1/N of the update's HBM
// traffic per rank, no per-tile signals (receivers need W' only at the end).
// warp 0: TMA producer, warp 1: storer, warps 2..15: fold (+ update)
constexpr int kPushConsumerBase = 64;
constexpr int kPushConsumerWarps = kArThreads / 32 - 2;

__device__ __forceinline__ void bulk_store_nc(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_addr(ssrc)), "r"(bytes)
               : "memory");
}
// 16-byte aligned slice j of an n-element buffer (the tail n & 3 is not in any)
__host__ __device__ __forceinline__ void push_slice(int64_t n, int N, int j, int64_t* lo,
                                                    int64_t* hi) {
  const int64_t n4 = n & ~int64_t(3);
  const int64_t per = ((n4 / 4 + N - 1) / N) * 4;
  const int64_t l = static_cast<int64_t>(j) * per, h = static_cast<int64_t>(j + 1) * per;
  *lo = l < n4 ? l : n4;
  *hi = h < n4 ? h : n4;
}

// Tile t of an owner slice [A, A + L): the first `nsmall` tiles (one per CTA)
// are a quarter of the full size, so every CTA's first fold -- and with it
// the first pushes -- needs a quarter of the bytes (the pipeline ramp keeps the
// push direction of the links idle until then).
struct PushTiles {
  int64_t A, L, TE, TEs, nsmall, T;
  __device__ PushTiles(int64_t a, int64_t b, int64_t te, int ctas) : A(a), L(b - a), TE(te) {
    TEs = max(int64_t(4), (te / 4) & ~int64_t(3));
    nsmall = min(static_cast<int64_t>(ctas), L / TEs);
    T = nsmall + (L - nsmall * TEs + TE - 1) / TE;
  }
  __device__ void span(int64_t t, int64_t* lo, int64_t* hi) const {
    *lo = t < nsmall ? A + t * TEs : A + nsmall * TEs + (t - nsmall) * TE;
    *hi = min(A + L, *lo + (t < nsmall ? TEs : TE));
  }
};

template <int kEpi>
__global__ void __launch_bounds__(kArThreads, 1)
    allreduce_push_kernel(const __grid_constant__ AllreduceArgs a) {
  constexpr bool kUpd = kEpi != 0;
  constexpr bool kMom = kEpi >= 3;
  const int view = blockIdx.x / a.ctas_per_view;
  const int local_cta = blockIdx.x % a.ctas_per_view;
  const ViewArgs& v = a.v[view];
  const int tid = threadIdx.x;
  const int N = a.n_ranks, me = v.rank;
  const int64_t TE = a.seg;
  const int S = a.lag;
  int64_t A, B;
  push_slice(a.n, N, me, &A, &B);
  const PushTiles tiles(A, B, TE, a.ctas_per_view);
  const int64_t T = tiles.T;
  const int64_t ulen = kUpd ? a.update_len : 0;  // a multiple of 4 (host)
  const size_t slot_f = static_cast<size_t>(TE);
  const int w_slot = N + 1, m_slot = N + 2;
  // [N rank slots][result g][W][momentum]
  const size_t stage_f = slot_f * (N + 1 + (kUpd ? (kMom ? 2 : 1) : 0));
  __shared__ uint32_t s_epoch;
  __shared__ __align__(8) uint64_t full[8], empty[8], folded[8];
  __shared__ int64_t s_tile[8];  // the tile a stage holds (-1: no more work)
  __shared__ FoldProg prog;
  extern __shared__ __align__(128) char ring[];
  float* ringf = reinterpret_cast<float*>(ring);
  for (int i = tid; i < static_cast<int>(sizeof(FoldProg) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(&prog)[i] = reinterpret_cast<const uint32_t*>(a.prog)[i];
  if (tid == 0) {
    s_epoch = *reinterpret_cast<volatile uint32_t*>(&v.ctrl->epoch) + 1;
    for (int st = 0; st < S; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 1);
      mbar_init(&folded[st], kPushConsumerWarps);
    }
    mbar_init_fence();
  }
  __syncthreads();
  const uint32_t epoch = s_epoch;
  int tn = 0;  // trace events (role 0: thread 0, role 1: storer, role 2: fold warp 0)
  if (tid == 0) trace_ev(a, 0, tn, EV_START, 0);
  const bool ok = entry_barrier(a, v, local_cta, epoch);
  if (tid == 0) trace_ev(a, 0, tn, EV_ENTRY, 0);
  if (ok) [&]() {
    if (tid < 32) {  // ---------------- producer (+ the buffer's tail) ----------------
      if (tid != 0) return;
      if (me == N - 1 && local_cta == 0) {
        // <= 3 elements past the last slice; update_len <= n & ~3 (host), so
        // these are plain sums in every mode
        for (int64_t i = a.n & ~int64_t(3); i < a.n; ++i) {
          float x[MD_MAX_RANKS];
          for (int r = 0; r < N; ++r) x[r] = r == me ? v.buf[i] : v.peer[r][i];
          const float g = fold_prog(prog.c[color_of(a.n, a.k, i)], x, 1, 0);
          for (int r = 0; r < N; ++r) (r == me ? v.buf : const_cast<float*>(v.peer[r]))[i] = g;
        }
        __threadfence_system();  // tail pushes are generic stores: visible before our done flag
      }
      fence_proxy_async_global();
      // tiles are handed out dynamically (a per-call counter in the own
      // control block, reset by the exit barrier): CTAs whose NVLink traffic
      // is served faster take more tiles, so all of them finish together
      // (static round-robin tiles measured a 115-240 us spread of CTA finish
      // times at N = 4, profiles/r02_trace_n4_sharded.json)
      for (uint32_t seq = 0;; ++seq) {
        const uint32_t st = seq % S;
        if (seq >= static_cast<uint32_t>(S)) {
          uint32_t spins = 0;
          while (!mbar_try_wait(&empty[st], ((seq / S) - 1) & 1))
            if ((++spins & 1023) == 0 && aborted(v)) return;
        }
        const int64_t t = atomicAdd(&v.ctrl->queue_head, 1u);
        if (t >= T) {  // no more work: a sentinel stage ends the consumers and the storer
          s_tile[st] = -1;
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&full[st])) : "memory");
          return;
        }
        s_tile[st] = t;
        int64_t lo, hi;
        tiles.span(t, &lo, &hi);
        const uint32_t bytes = static_cast<uint32_t>((hi - lo) * 4);
        const int64_t whi = min(hi, ulen);
        const uint32_t wbytes = whi > lo ? static_cast<uint32_t>((whi - lo) * 4) : 0u;
        float* stage = ringf + st * stage_f;
        mbar_expect_tx(&full[st], bytes * N + wbytes * (kMom ? 2 : 1));
        for (int r = 0; r < N; ++r)
          tma_load_1d(stage + r * slot_f, (r == me ? v.buf : v.peer[r]) + lo, bytes, &full[st]);
        if (kUpd && wbytes) {
          tma_load_1d(stage + w_slot * slot_f, v.w + lo, wbytes, &full[st]);
          if (kMom) tma_load_1d(stage + m_slot * slot_f, v.mom + lo, wbytes, &full[st]);
        }
      }
    } else if (tid < kPushConsumerBase) {  // ---------------- storer ----------------
      if (tid != 32) return;
      uint32_t seq = 0;
      int sn = 0;
      for (;; ++seq) {
        const uint32_t st = seq % S;
        uint32_t spins = 0;
        while (!mbar_try_wait(&folded[st], (seq / S) & 1))
          if ((++spins & 1023) == 0 && aborted(v)) return;
        const int64_t t = s_tile[st];
        if (t < 0) break;
        if (seq == 0) trace_ev(a, 1, sn, EV_FIRST, 0);
        int64_t lo, hi;
        tiles.span(t, &lo, &hi);
        const uint32_t bytes = static_cast<uint32_t>((hi - lo) * 4);
        const float* stage = ringf + st * stage_f;
        const float* res = stage + N * slot_f;
        if (kUpd) {
          const int64_t whi = min(hi, ulen);
          if (whi > lo) {  // W' to every rank (own last: peers' pushes first on the wire)
            const uint32_t wb = static_cast<uint32_t>((whi - lo) * 4);
            for (int q = 0; q < N; ++q) {
              const int r = (me + 1 + q) % N;
              bulk_store_nc((r == me ? v.w : v.peer_w[r]) + lo, stage + w_slot * slot_f, wb);
            }
            if (kMom) bulk_store_nc(v.mom + lo, stage + m_slot * slot_f, wb);
          }
          const int64_t glo = max(lo, whi);
          if (hi > glo)  // past the update range: g to every peer, as a plain call
            for (int q = 0; q < N - 1; ++q) {
              const int r = (me + 1 + q) % N;
              bulk_store_nc(const_cast<float*>(v.peer[r]) + glo, res + (glo - lo),
                            static_cast<uint32_t>((hi - glo) * 4));
            }
          bulk_store_nc(v.buf + lo, res, bytes);  // g: the own slice only
        } else {
          for (int q = 0; q < N; ++q) {  // own buffer last: peers' pushes first on the wire
            const int r = (me + 1 + q) % N;
            bulk_store_nc((r == me ? v.buf : const_cast<float*>(v.peer[r])) + lo, res, bytes);
          }
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (seq >= 1) {  // the previous tile's stores have read their SMEM: free its stage
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&empty[(seq - 1) % S]))
                       : "memory");
        }
      }
      trace_ev(a, 1, sn, EV_ISSUED, static_cast<int>(seq));
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // every push has landed
      trace_ev(a, 1, sn, EV_DONE, static_cast<int>(seq));
    } else {  // ---------------- fold (+ the slice's SGD update) ----------------
      const int ct = tid - kPushConsumerBase, nct = kPushConsumerWarps * 32;
      for (uint32_t seq = 0;; ++seq) {
        const uint32_t st = seq % S;
        uint32_t spins = 0;
        while (!mbar_try_wait(&full[st], (seq / S) & 1))
          if ((++spins & 1023) == 0 && aborted(v)) return;
        const int64_t t = s_tile[st];
        if (t < 0) {  // pass the sentinel on to the storer
          __syncwarp();
          if ((ct & 31) == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&folded[st])) : "memory");
          return;
        }
        float* stage = ringf + st * stage_f;
        float* res = stage + N * slot_f;
        int64_t lo, hi;
        tiles.span(t, &lo, &hi);
        const int64_t len = hi - lo;
        const int64_t wlen = kUpd ? max(int64_t(0), min(len, ulen - lo)) : 0;
        for (int64_t e = 4 * ct; e < len; e += 4 * nct) {
          const int c0 = color_of(a.n, a.k, lo + e);
          float4 g;
          if (color_of(a.n, a.k, lo + e + 3) == c0) {
            g = fold_prog4(prog.c[c0], stage, slot_f, e);
          } else {
            g.x = fold_prog(prog.c[c0], stage, slot_f, e);
            g.y = fold_prog(prog.c[color_of(a.n, a.k, lo + e + 1)], stage, slot_f, e + 1);
            g.z = fold_prog(prog.c[color_of(a.n, a.k, lo + e + 2)], stage, slot_f, e + 2);
            g.w = fold_prog(prog.c[color_of(a.n, a.k, lo + e + 3)], stage, slot_f, e + 3);
          }
          *reinterpret_cast<float4*>(res + e) = g;
          if constexpr (kUpd) {
            if (e < wlen) {  // wlen is a multiple of 4
              float4* wp = reinterpret_cast<float4*>(stage + w_slot * slot_f + e);
              float4* mp = reinterpret_cast<float4*>(stage + m_slot * slot_f + e);
              float4 w = *wp;
              float4 m = kMom ? *mp : make_float4(0.f, 0.f, 0.f, 0.f);
              sgd_elem<kEpi>(w.x, g.x, m.x, a);
              sgd_elem<kEpi>(w.y, g.y, m.y, a);
              sgd_elem<kEpi>(w.z, g.z, m.z, a);
              sgd_elem<kEpi>(w.w, g.w, m.w, a);
              *wp = w;
              if (kMom) *mp = m;
            }
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // SMEM -> bulk-store reads
        __syncwarp();
        if ((ct & 31) == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&folded[st])) : "memory");
      }
    }
  }();
  exit_barrier(a, v, epoch);
}

struct TraceBuf {
  void* ptr = nullptr;
  size_t bytes = 0, used = 0;
};
static TraceBuf g_trace[64];

// ---- plan construction (host) ------------------------------------------------
static int build_rank_plans(int n, int k, const int32_t* parent, const int32_t* child_ptr,
                            const int32_t* child_idx, const int32_t* self_pos,
                            std::vector<RankPlan>* out) {
  out->assign(n, RankPlan{});
  for (int c = 0; c < k; ++c) {
    const int32_t* par = parent + c * n;
    int root = -1;
    for (int r = 0; r < n; ++r) {
      if (par[r] < -1 || par[r] >= n || par[r] == r) {
        set_error("color %d: bad parent %d of rank %d", c, par[r], r);
        return MD_ERR_INVALID_CONFIG;
      }
      if (par[r] == -1) {
        if (root >= 0) {
          set_error("color %d has two roots (%d, %d)", c, root, r);
          return MD_ERR_INVALID_CONFIG;
        }
        root = r;
      }
    }
    if (root < 0) {
      set_error("color %d has no root", c);
      return MD_ERR_INVALID_CONFIG;
    }
    auto kids = [&](int r, int* cnt) {
      int row = c * n + r;
      *cnt = child_ptr[row + 1] - child_ptr[row];
      return child_idx + child_ptr[row];
    };
    // consistency + acyclicity: depth via parent chain (<= n steps)
    std::vector<int> depth(n, -1), height(n, 0);
    for (int r = 0; r < n; ++r) {
      int d = 0, cur = r;
      while (par[cur] >= 0 && d <= n) {
        cur = par[cur];
        ++d;
      }
      if (d > n || cur != root) {
        set_error("color %d: cycle reachable from rank %d", c, r);
        return MD_ERR_INVALID_CONFIG;
      }
      depth[r] = d;
      int cnt;
      const int32_t* ch = kids(r, &cnt);
      if (cnt < 0 || cnt > MD_MAX_RANKS) {
        set_error("color %d: rank %d has %d children", c, r, cnt);
        return MD_ERR_INVALID_CONFIG;
      }
      for (int j = 0; j < cnt; ++j) {
        if (ch[j] < 0 || ch[j] >= n || par[ch[j]] != r) {
          set_error("color %d: child %d of %d disagrees with parent map", c, ch[j], r);
          return MD_ERR_INVALID_CONFIG;
        }
      }
    }
    int total_children = 0;
    for (int r = 0; r < n; ++r) {
      int cnt;
      kids(r, &cnt);
      total_children += cnt;
    }
    if (total_children != n - 1) {
      set_error("color %d: children lists cover %d ranks, expected %d", c, total_children, n - 1);
      return MD_ERR_INVALID_CONFIG;
    }
    // heights, deepest first
    std::vector<int> order(n);
    for (int r = 0; r < n; ++r) order[r] = r;
    std::sort(order.begin(), order.end(), [&](int x, int y) { return depth[x] > depth[y]; });
    for (int r : order)
      if (par[r] >= 0) height[par[r]] = std::max(height[par[r]], height[r] + 1);
    const int H = height[root];

    auto fold_pos = [&](int r) { return self_pos ? self_pos[c * n + r] : 0; };
    for (int r = 0; r < n; ++r) {
      RankPlan& rp = (*out)[r];
      int cnt;
      const int32_t* ch = kids(r, &cnt);
      int sp = fold_pos(r);
      if (sp < 0 || sp > cnt) {
        set_error("color %d: self position %d out of range for rank %d", c, sp, r);
        return MD_ERR_INVALID_CONFIG;
      }
      Task up{};
      up.type = 0;
      up.color = c;
      up.stage = height[r];
      up.parent = par[r];
      up.is_leaf = cnt == 0;
      up.n_fold = cnt + 1;
      for (int j = 0, q = 0; j <= cnt; ++j) {
        if (j == sp) {
          up.fold_src[j] = r;
          up.fold_leaf[j] = 0;
        } else {
          int chr = ch[q++];
          up.fold_src[j] = chr;
          int gc;
          kids(chr, &gc);
          up.fold_leaf[j] = gc == 0;
        }
      }
      if (par[r] >= 0) {
        int pcnt;
        const int32_t* pch = kids(par[r], &pcnt);
        int ci = 0;
        while (ci < pcnt && pch[ci] != r) ++ci;
        int psp = fold_pos(par[r]);
        up.my_slot = ci >= psp ? ci + 1 : ci;
      } else {
        up.n_down = cnt;
        for (int j = 0; j < cnt; ++j) up.down[j] = ch[j];
      }
      rp.t[rp.n_tasks++] = up;
      if (par[r] >= 0) {
        Task dn{};
        dn.type = 1;
        dn.color = c;
        dn.stage = H + depth[r];
        dn.parent = par[r];
        dn.n_down = cnt;
        for (int j = 0; j < cnt; ++j) dn.down[j] = ch[j];
        rp.t[rp.n_tasks++] = dn;
      }
    }
  }
  for (auto& rp : *out)
    std::stable_sort(rp.t, rp.t + rp.n_tasks,
                     [](const Task& x, const Task& y) { return x.stage < y.stage; });
  return MD_OK;
}

// Each color's fold as a post-order program over rank slots (ColorProg), from
// the same per-rank UP tasks the tree schedule runs: op = (folding rank, its
// fold list), ordered by subtree height so children come before parents.
static void build_fold_prog(const std::vector<RankPlan>& plans, int n, int k, FoldProg* out) {
  memset(out, 0, sizeof(*out));
  for (int c = 0; c < k; ++c) {
    ColorProg& p = out->c[c];
    std::vector<std::pair<int, const Task*>> ops;  // (folding rank, its UP task)
    for (int r = 0; r < n; ++r)
      for (int i = 0; i < plans[r].n_tasks; ++i) {
        const Task& t = plans[r].t[i];
        if (t.type != 0 || t.color != c) continue;
        if (t.parent < 0) p.root = static_cast<uint8_t>(r);
        if (t.n_fold > 1) ops.push_back({r, &t});
      }
    std::stable_sort(ops.begin(), ops.end(), [](const auto& x, const auto& y) {
      return x.second->stage < y.second->stage;
    });
    int off = 0;
    for (const auto& [r, t] : ops) {
      p.op_dst[p.n_ops] = static_cast<uint8_t>(r);
      p.op_cnt[p.n_ops] = static_cast<uint8_t>(t->n_fold);
      for (int j = 0; j < t->n_fold; ++j) p.items[off++] = static_cast<uint8_t>(t->fold_src[j]);
      ++p.n_ops;
    }
  }
}

// Owner-computes schedule ("which data movement"): the
// buffer is cut into n equal slices (chunk_of with n "colors"); rank j owns
// slice j: it pulls every rank's slice j and evaluates each element's OWN
// color fold program (task type 2), then every other rank copies the final
// slice from j (DOWN). Same adds in the same order per element as the tree
// schedule -- same bits -- but every rank ingests 2 (n-1)/n of the buffer for
// any k, where the reference's trees cap k = 1 / 2 at N = 4 at 50 / 75 %.
static void build_owner_plans(int n, std::vector<RankPlan>* out) {
  out->assign(n, RankPlan{});
  for (int j = 0; j < n; ++j) {
    for (int r = 0; r < n; ++r) {
      RankPlan& rp = (*out)[r];
      Task t{};
      t.color = j;
      if (r == j) {
        t.type = 2;
        t.stage = 0;
        t.parent = -1;
        t.n_fold = n;
        for (int q = 0; q < n; ++q) {
          t.fold_src[q] = q;
          t.fold_leaf[q] = 1;  // raw inputs: ready at the entry barrier
        }
        t.n_down = n - 1;
        for (int q = 0, c = 0; q < n; ++q)
          if (q != j) t.down[c++] = q;
      } else {
        t.type = 1;
        t.stage = 1;
        t.parent = j;
        t.n_down = 0;
      }
      rp.t[rp.n_tasks++] = t;
    }
  }
  for (auto& rp : *out)
    std::stable_sort(rp.t, rp.t + rp.n_tasks,
                     [](const Task& x, const Task& y) { return x.stage < y.stage; });
}

}  // namespace md

using namespace md;

extern "C" {

int md_device_count(int* n) {
  MD_CUDA_TRY(cudaGetDeviceCount(n));
  return MD_OK;
}

int md_enable_peer_access(int dev, int peer) {
  if (dev == peer) return MD_OK;
  int prev;
  MD_CUDA_TRY(cudaGetDevice(&prev));
  MD_CUDA_TRY(cudaSetDevice(dev));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    e = cudaSuccess;
  }
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    set_error("cudaDeviceEnablePeerAccess(%d -> %d): %s", dev, peer, cudaGetErrorString(e));
    return MD_ERR_CUDA;
  }
  return MD_OK;
}

typedef int (*PFN_getAddressRange)(unsigned long long*, size_t*, unsigned long long);

int md_mem_export(const void* ptr, unsigned char handle[MD_IPC_HANDLE_BYTES], uint64_t* offset) {
  static PFN_getAddressRange fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    MD_CUDA_TRY(cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q));
    if (!p) {
      set_error("cuMemGetAddressRange unavailable");
      return MD_ERR_CUDA;
    }
    fn = reinterpret_cast<PFN_getAddressRange>(p);
  }
  unsigned long long base = 0;
  size_t size = 0;
  int rc = fn(&base, &size, reinterpret_cast<unsigned long long>(ptr));
  if (rc != 0) {
    set_error("cuMemGetAddressRange failed (%d)", rc);
    return MD_ERR_CUDA;
  }
  cudaIpcMemHandle_t h;
  MD_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  static_assert(sizeof(h) == MD_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle, &h, sizeof(h));
  *offset = reinterpret_cast<unsigned long long>(ptr) - base;
  return MD_OK;
}

int md_mem_import(const unsigned char handle[MD_IPC_HANDLE_BYTES], void** base) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  MD_CUDA_TRY(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
  return MD_OK;
}

int md_mem_close(void* base) {
  MD_CUDA_TRY(cudaIpcCloseMemHandle(base));
  return MD_OK;
}

int md_comm_create(int32_t rank, int32_t n_ranks, int32_t device, md_comm_t** out) {
  if (n_ranks < 1 || n_ranks > MD_MAX_RANKS || rank < 0 || rank >= n_ranks) {
    set_error("rank %d of %d unsupported (max %d ranks)", rank, n_ranks, MD_MAX_RANKS);
    return MD_ERR_INVALID_CONFIG;
  }
  int prev;
  MD_CUDA_TRY(cudaGetDevice(&prev));
  MD_CUDA_TRY(cudaSetDevice(device));
  md_comm* c = new md_comm();
  c->rank = rank;
  c->n_ranks = n_ranks;
  c->device = device;
  c->epoch = 0;
  c->timeout_s = 30.0;
  cudaError_t e = cudaMalloc(&c->ctrl, sizeof(Ctrl));
  if (e == cudaSuccess) e = cudaMemset(c->ctrl, 0, sizeof(Ctrl));
  if (e == cudaSuccess) e = cudaHostAlloc(&c->err_host, 2 * sizeof(int32_t), cudaHostAllocMapped);
  if (e == cudaSuccess) {
    c->err_host[0] = c->err_host[1] = 0;
    e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->err_dev), c->err_host, 0);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    set_error("md_comm_create: %s", cudaGetErrorString(e));
    delete c;
    return MD_ERR_CUDA;
  }
  for (int r = 0; r < MD_MAX_RANKS; ++r) c->peer_ctrl[r] = nullptr;
  c->peer_ctrl[rank] = c->ctrl;
  *out = c;
  return MD_OK;
}

int md_comm_destroy(md_comm_t* c) {
  if (!c) return MD_OK;
  int prev;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  cudaFree(c->ctrl);
  cudaFreeHost(c->err_host);
  cudaSetDevice(prev);
  delete c;
  return MD_OK;
}

int md_comm_ctrl_ptr(md_comm_t* c, void** ctrl) {
  *ctrl = c->ctrl;
  return MD_OK;
}

int md_comm_set_peer_ctrl(md_comm_t* c, void* const* ptrs, int32_t n) {
  if (n != c->n_ranks) {
    set_error("expected %d control pointers, got %d", c->n_ranks, n);
    return MD_ERR_INVALID_CONFIG;
  }
  for (int r = 0; r < n; ++r)
    c->peer_ctrl[r] = (r == c->rank) ? c->ctrl : static_cast<Ctrl*>(ptrs[r]);
  return MD_OK;
}

int md_comm_take_error(md_comm_t* c, int32_t* code, int32_t* detail) {
  volatile int32_t* e = c->err_host;
  *code = e[0];
  *detail = e[1];
  e[0] = 0;
  e[1] = 0;
  return MD_OK;
}

int md_comm_set_timeout(md_comm_t* c, double seconds) {
  if (!(seconds > 0)) {
    set_error("timeout must be > 0");
    return MD_ERR_INVALID_CONFIG;
  }
  c->timeout_s = seconds;
  return MD_OK;
}

int md_plan_create(int32_t n_ranks, int32_t k, const int32_t* parent, const int32_t* child_ptr,
                   const int32_t* child_idx, const int32_t* self_pos, int32_t device,
                   md_plan_t** out) {
  if (n_ranks < 1 || n_ranks > MD_MAX_RANKS) {
    set_error("n_ranks %d unsupported (max %d)", n_ranks, MD_MAX_RANKS);
    return MD_ERR_INVALID_CONFIG;
  }
  if (k < 1 || k > MD_MAX_COLORS) {
    set_error("%d colors unsupported (max %d)", k, MD_MAX_COLORS);
    return MD_ERR_INVALID_CONFIG;
  }
  std::vector<RankPlan> host;
  int rc = build_rank_plans(n_ranks, k, parent, child_ptr, child_idx, self_pos, &host);
  if (rc != MD_OK) return rc;
  int prev;
  MD_CUDA_TRY(cudaGetDevice(&prev));
  MD_CUDA_TRY(cudaSetDevice(device));
  md_plan* p = new md_plan();
  p->n_ranks = n_ranks;
  p->k = k;
  p->device = device;
  p->host = host;
  p->prog_dev = nullptr;
  p->owner_dev = nullptr;
  p->schedule = MD_SCHED_TREE;
  p->route = MD_ROUTE_AUTO;
  p->tile = 0;
  FoldProg prog;
  build_fold_prog(host, n_ranks, k, &prog);
  build_owner_plans(n_ranks, &p->owner_host);
  cudaError_t e = cudaMalloc(&p->dev, sizeof(RankPlan) * n_ranks);
  if (e == cudaSuccess)
    e = cudaMemcpy(p->dev, host.data(), sizeof(RankPlan) * n_ranks, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&p->prog_dev, sizeof(FoldProg));
  if (e == cudaSuccess) e = cudaMemcpy(p->prog_dev, &prog, sizeof(FoldProg), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&p->owner_dev, sizeof(RankPlan) * n_ranks);
  if (e == cudaSuccess)
    e = cudaMemcpy(p->owner_dev, p->owner_host.data(), sizeof(RankPlan) * n_ranks,
                   cudaMemcpyHostToDevice);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    set_error("md_plan_create: %s", cudaGetErrorString(e));
    delete p;
    return MD_ERR_CUDA;
  }
  *out = p;
  return MD_OK;
}

int md_plan_set_schedule(md_plan_t* p, int32_t schedule) {
  if (!p || (schedule != MD_SCHED_TREE && schedule != MD_SCHED_OWNER)) {
    set_error("bad plan or schedule %d", schedule);
    return MD_ERR_INVALID_CONFIG;
  }
  p->schedule = schedule;
  return MD_OK;
}

int md_plan_set_route(md_plan_t* p, int32_t route, int64_t tile) {
  if (!p || route < MD_ROUTE_AUTO || route > MD_ROUTE_PUSH || tile < 0) {
    set_error("bad plan, route %d or tile %lld", route, (long long)tile);
    return MD_ERR_INVALID_CONFIG;
  }
  p->route = route;
  p->tile = tile & ~int64_t(3);
  return MD_OK;
}

int md_plan_destroy(md_plan_t* p) {
  if (!p) return MD_OK;
  int prev;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  cudaFree(p->dev);
  cudaFree(p->prog_dev);
  cudaFree(p->owner_dev);
  cudaSetDevice(prev);
  delete p;
  return MD_OK;
}

}  // extern "C"

namespace {
using namespace md;

// Routing knobs, read ONCE per process (the environment is for tools and A/B
// runs; tests and callers pick routes per plan with md_plan_set_route).
struct ArEnv {
  int64_t ll_max = -1;       // MD_AR_LL_MAX: largest LL buffer (bytes), -1 = built-in
  int64_t oneshot_max = -1;  // MD_AR_ONESHOT_MAX
  int32_t route = MD_ROUTE_AUTO;  // MD_AR_ROUTE=tree|queue|ll|oneshot|stream|push
  int64_t tile = 0;          // MD_AR_TILE: tile of the tiled routes (elements)
  int32_t lag = -1;          // MD_AR_LAG: queue kernel pipeline lag
  bool trace = false;        // MD_AR_TRACE=1: per-CTA event log (md_trace_dump)
  bool sys_fence = false;    // MD_AR_SYS_FENCE=1: system-scope release for every flag
};

const ArEnv& ar_env() {
  static const ArEnv env = [] {
    ArEnv e;
    if (const char* x = getenv("MD_AR_LL_MAX")) e.ll_max = atoll(x);
    if (const char* x = getenv("MD_AR_ONESHOT_MAX")) e.oneshot_max = atoll(x);
    if (const char* x = getenv("MD_AR_TILE")) e.tile = std::max<int64_t>(0, atoll(x)) & ~int64_t(3);
    if (const char* x = getenv("MD_AR_LAG")) e.lag = std::max(0, atoi(x));
    e.trace = getenv("MD_AR_TRACE") != nullptr;
    e.sys_fence = getenv("MD_AR_SYS_FENCE") != nullptr;
    if (const char* x = getenv("MD_AR_ROUTE")) {
      static const char* names[] = {"auto", "tree", "queue", "ll", "oneshot", "stream", "push"};
      for (int r = 0; r <= MD_ROUTE_PUSH; ++r)
        if (!strcmp(x, names[r])) e.route = r;
    }
    return e;
  }();
  return env;
}

// Smallest plain buffer (bytes) the owner-push kernel takes by default.
// Measured against every other route (graph-timed C2 sweep, round 2,
// profiles/r02_sweep_n{2,4}.csv): N = 2 push 22.3 us at 4 MiB (one-shot 23.0)
// and 42.0 us at 16 MiB (tree 45.9-61.6), LL stays faster at 1 MiB (10.4 vs
// 17.9); N = 4 push 19.3 us at 1 MiB (LL 20.6-20.9) and faster at every size
// above.
int64_t push_min_bytes(int N) { return N == 2 ? (int64_t(4) << 20) : (int64_t(1) << 20); }

// Pipeline segment cap for a color chunk of `chunk` elements: about two
// segments per SM, never below 4096 elements (the per-segment flag cost).
// segment_elems is an upper bound only -- the bits never depend on it
// (pkg/tests/test_collectives.py:131-147). Measured at N = 4, k = 4: 4 MiB
// 38.3 -> 35.3 us, 16 MiB 65.9 -> 62 us; 100 MB unchanged (16384 stays).
int64_t auto_seg(int64_t chunk, int dev) {
  const int64_t want = (chunk / (2 * static_cast<int64_t>(sm_count(dev))) + 3) & ~int64_t(3);
  return std::max<int64_t>(4096, want);
}

// Largest buffer (bytes) the one-shot kernel takes at world size N: at N = 2
// its ingress equals the tree's, so any size that fits; above, it pulls
// (N-1) x bytes against the tree's 2 (N-1)/N x bytes, so only latency-bound
// sizes (measured crossover, profiles/README.md).
int64_t oneshot_max_bytes(int N) {
  if (ar_env().oneshot_max >= 0) return ar_env().oneshot_max;
  return N == 2 ? (int64_t(1) << 40) : (int64_t(1) << 20);
}

// Smallest buffer (bytes) a replicated fused N = 2 call streams (measured win
// at the 102.4 MB C5 buffer; below that the tree keeps it).
constexpr int64_t kStreamMinBytes = int64_t(64) << 20;

// Largest buffer (bytes) the LL push kernel takes: it moves 2 x (N-1) x bytes
// out of every rank (value + epoch words), so only latency-bound sizes:
// measured faster than the one-shot pull up to 1 MiB at N = 2 and 4 (10.4 vs
// 15.9 us and 20.0 vs 21.3 us), untested above N = 4 (256 KiB there).
int64_t ll_max_bytes(int N) {
  if (ar_env().ll_max >= 0) return ar_env().ll_max;
  return N <= 4 ? (int64_t(1) << 20) : (int64_t(256) << 10);
}

// diagnostics (MD_AR_TRACE=1): the per-CTA event log of this call, one per device
int setup_trace(AllreduceArgs* a, int dev, int ctas, int n_views) {
  a->trace = nullptr;
  if (!ar_env().trace || dev < 0 || dev >= 64) return MD_OK;
  const size_t bytes = sizeof(TraceEv) * 3 * kTraceHalf * static_cast<size_t>(ctas) * n_views;
  if (!g_trace[dev].ptr || g_trace[dev].bytes < bytes) {
    if (g_trace[dev].ptr) cudaFree(g_trace[dev].ptr);
    MD_CUDA_TRY(cudaMalloc(&g_trace[dev].ptr, bytes));
    MD_CUDA_TRY(cudaMemset(g_trace[dev].ptr, 0, bytes));
    g_trace[dev].bytes = bytes;
  }
  // (md_trace_dump re-zeroes the log, so a traced call adds no work of its own)
  g_trace[dev].used = bytes;
  a->trace = static_cast<TraceEv*>(g_trace[dev].ptr);
  return MD_OK;
}

// cudaFuncSetAttribute(max dynamic SMEM) once per (kernel, device)
int smem_attr_once(const void* k, int dev, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  std::lock_guard<std::mutex> g(mu);
  for (const auto& d : done)
    if (d.first == k && d.second == dev) return MD_OK;
  MD_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(bytes)));
  done.emplace_back(k, dev);
  return MD_OK;
}

// Emulated ranks (n_views > 1) wait on each other's CTAs on ONE device: a
// cooperative launch guarantees they are co-resident. A real rank's CTAs only
// wait on other GPUs (never on a sibling CTA), so a plain launch of <= one
// CTA per SM is deadlock-free there.
int launch_views(const void* k, unsigned grid, int n_views, size_t smem, AllreduceArgs* a,
                 void* stream) {
  void* args[] = {a};
  if (n_views > 1) {
    MD_CUDA_TRY(cudaLaunchCooperativeKernel(k, dim3(grid * n_views), dim3(kArThreads), args, smem,
                                            as_stream(stream)));
  } else {
    MD_CUDA_TRY(cudaLaunchKernel(k, dim3(grid), dim3(kArThreads), args, smem, as_stream(stream)));
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return MD_OK;
}

#define MD_EPI_TABLE(kernel)                                                                   \
  static const void* kernel##_of(int epi) {                                                    \
    switch (epi) {                                                                             \
      case 1: return reinterpret_cast<const void*>(kernel<1>);                                 \
      case 2: return reinterpret_cast<const void*>(kernel<2>);                                 \
      case 3: return reinterpret_cast<const void*>(kernel<3>);                                 \
      case 4: return reinterpret_cast<const void*>(kernel<4>);                                 \
      default: return reinterpret_cast<const void*>(kernel<0>);                                \
    }                                                                                          \
  }
MD_EPI_TABLE(allreduce_ll_kernel)
MD_EPI_TABLE(allreduce_oneshot_kernel)
MD_EPI_TABLE(allreduce_stream_kernel)
MD_EPI_TABLE(allreduce_push_kernel)
MD_EPI_TABLE(allreduce_channels_kernel)
MD_EPI_TABLE(allreduce_kernel)
#undef MD_EPI_TABLE

std::atomic<uint64_t> g_last_route[64];

void record_route(int dev, int route, int64_t tile, bool sharded) {
  if (dev >= 0 && dev < 64)
    g_last_route[dev].store(static_cast<uint64_t>(route) | (sharded ? 0x80u : 0u) |
                                (static_cast<uint64_t>(tile) << 8),
                            std::memory_order_relaxed);
}

uint64_t cfg_word_of(int route, bool owner_sched, bool sharded, int64_t geometry) {
  return static_cast<uint64_t>(route) | (static_cast<uint64_t>(owner_sched) << 4) |
         (static_cast<uint64_t>(sharded) << 5) | (static_cast<uint64_t>(geometry) << 8);
}

}  // namespace

extern "C" {

int md_last_route(int32_t device, int32_t* route, int64_t* tile, int32_t* sharded) {
  if (device < 0 || device >= 64) {
    set_error("bad device %d", device);
    return MD_ERR_INVALID_CONFIG;
  }
  const uint64_t w = g_last_route[device].load(std::memory_order_relaxed);
  if (route) *route = static_cast<int32_t>(w & 0x7f);
  if (sharded) *sharded = (w & 0x80) ? 1 : 0;
  if (tile) *tile = static_cast<int64_t>(w >> 8);
  return MD_OK;
}

int md_allreduce(md_comm_t* const* comms, int32_t n_views, const md_plan_t* plan,
                 float* const* bufs, int64_t n, const float* const* workers, int32_t n_workers,
                 float* const* w, float* const* mom, int64_t update_len, float c, float mu,
                 float wd_b, int64_t seg_elems, int32_t ctas, void* stream) {
  md_update_t u{w, mom, update_len, c, mu, wd_b, MD_UPDATE_REPLICATED};
  return md_allreduce_ex(comms, n_views, plan, bufs, n, workers, n_workers, w ? &u : nullptr,
                         seg_elems, ctas, stream);
}

int md_allreduce_ex(md_comm_t* const* comms, int32_t n_views, const md_plan_t* plan,
                    float* const* bufs, int64_t n, const float* const* workers, int32_t n_workers,
                    const md_update_t* upd, int64_t seg_elems, int32_t ctas, void* stream) {
  if (!plan || n_views < 1 || n_views > MD_MAX_RANKS) {
    set_error("bad plan/view count");
    return MD_ERR_INVALID_CONFIG;
  }
  const int N = plan->n_ranks;
  const ArEnv& env = ar_env();
  if (n < 0) {
    set_error("negative length");
    return MD_ERR_INVALID_CONFIG;
  }
  if (n_workers < 0 || n_workers > MD_MAX_WORKERS || (n_workers > 0 && !workers)) {
    set_error("bad worker count %d (max %d)", n_workers, MD_MAX_WORKERS);
    return MD_ERR_INVALID_CONFIG;
  }
  if (seg_elems < 1) {
    set_error("segment_elems must be >= 1, got %lld", (long long)seg_elems);
    return MD_ERR_INVALID_CONFIG;
  }
  const bool has_update = upd != nullptr && upd->w != nullptr;
  const int64_t update_len = has_update ? upd->len : 0;
  if (has_update && (update_len < 0 || update_len > n)) {
    set_error("update_len %lld outside [0, %lld]", (long long)update_len, (long long)n);
    return MD_ERR_LENGTH_MISMATCH;
  }
  if (has_update && upd->mode != MD_UPDATE_REPLICATED && upd->mode != MD_UPDATE_SHARDED) {
    set_error("bad update mode %d", upd->mode);
    return MD_ERR_INVALID_CONFIG;
  }
  const bool mode_sharded = has_update && upd->mode == MD_UPDATE_SHARDED;
  const float c = has_update ? upd->c : 0.f, mu = has_update ? upd->mu : 0.f;
  const float wd_b = has_update ? upd->wd_b : 0.f;
  int dev;
  MD_CUDA_TRY(cudaGetDevice(&dev));
  AllreduceArgs a;
  memset(&a, 0, sizeof(a));
  a.plan = plan->dev;
  a.n = n;
  a.n_ranks = N;
  a.k = plan->k;
  a.n_views = n_views;
  a.n_workers = n_workers;
  a.has_update = has_update;
  a.update_len = update_len;
  a.c = c;
  a.mu = mu;
  a.wd_b = wd_b;
  a.flag_gpu_fence = !env.sys_fence;  // see publish_flags
  a.reverse_local = 1;
  a.prog = plan->prog_dev;
  a.prog_k = plan->k;
  // segment length: multiple of 4 elements, <= kMaxSegs segments per color
  const int64_t maxlen = (n + plan->k - 1) / plan->k;
  int64_t seg = std::max<int64_t>(4, (seg_elems + 3) & ~int64_t(3));
  if (N > 1) seg = std::min(seg, auto_seg(maxlen, dev));
  const int64_t min_seg = ((maxlen + 3) / kMaxSegs + 4 + 3) & ~int64_t(3);
  if (seg < min_seg) seg = min_seg;
  a.seg = seg;
  int64_t mx = 0;
  for (int col = 0; col < plan->k; ++col) {
    int64_t st, ln;
    chunk_of(n, plan->k, col, &st, &ln);
    mx = std::max(mx, nseg_of(st, ln, seg));
  }
  a.max_nseg = static_cast<int32_t>(mx);
  uintptr_t bits = 0;
  double timeout = 30.0;
  for (int vi = 0; vi < n_views; ++vi) {
    md_comm* cm = comms[vi];
    if (!cm || cm->n_ranks != N) {
      set_error("communicator/plan world size mismatch (%d vs %d)", cm ? cm->n_ranks : -1, N);
      return MD_ERR_INVALID_CONFIG;
    }
    ViewArgs& v = a.v[vi];
    v.rank = cm->rank;
    v.ctrl = cm->ctrl;
    for (int r = 0; r < N; ++r) {
      if (!cm->peer_ctrl[r]) {
        set_error("rank %d: control block of peer %d not installed", cm->rank, r);
        return MD_ERR_INVALID_CONFIG;
      }
      v.peer_ctrl[r] = cm->peer_ctrl[r];
      v.peer[r] = bufs[vi * N + r];
      bits |= reinterpret_cast<uintptr_t>(v.peer[r]);
    }
    v.buf = bufs[vi * N + cm->rank];
    for (int j = 0; j < n_workers; ++j) {
      v.workers[j] = workers[vi * n_workers + j];
      bits |= reinterpret_cast<uintptr_t>(v.workers[j]);
    }
    if (has_update) {
      // sharded: w holds every rank's (peer-mapped) weights, view-major
      v.w = mode_sharded ? upd->w[vi * N + cm->rank] : upd->w[vi];
      if (mode_sharded)
        for (int r = 0; r < N; ++r) {
          v.peer_w[r] = upd->w[vi * N + r];
          bits |= reinterpret_cast<uintptr_t>(v.peer_w[r]);
        }
      v.mom = (upd->mom && mu != 0.f) ? upd->mom[vi] : nullptr;
      bits |= reinterpret_cast<uintptr_t>(v.w) | reinterpret_cast<uintptr_t>(v.mom);
    }
    v.err = cm->err_dev;
    ++cm->epoch;
    timeout = std::min(timeout, cm->timeout_s);
  }
  a.vec_ok = (bits & 15) == 0;
  a.timeout_ns = static_cast<unsigned long long>(timeout * 1e9);
  const int req = plan->route != MD_ROUTE_AUTO ? plan->route : env.route;
  const int64_t tile_req = plan->tile ? plan->tile : env.tile;
  const bool auto_route = req == MD_ROUTE_AUTO;
  const int avail = sm_count(dev) / n_views;  // CTAs (one per SM) per view
  const bool fold_ok = N > 1 && n > 0 && n_workers == 0 && a.vec_ok && plan->prog_dev;

  // One rank, no worker fold: the collective is the identity and the call is
  // only its fused SGD update -- the streaming md_sgd_update kernel (8 CTAs x
  // 256 threads per SM) measured 82 vs 91 us for the 25.6M-float momentum +
  // weight-decay update (95 % vs 86 % of the HBM copy peak); same sgd1 math.
  if (N == 1 && n_views == 1 && n_workers == 0) {
    record_route(dev, MD_ROUTE_LOCAL, 0, false);
    if (!has_update || update_len == 0) return MD_OK;
    return md_sgd_update(a.v[0].w, a.v[0].buf, a.v[0].mom, update_len, c,
                         a.v[0].mom ? mu : 0.f, wd_b, stream);
  }
  int epi = 0;
  if (has_update) epi = (a.v[0].mom ? 3 : 1) + (wd_b != 0.f ? 1 : 0);

  // ---- owner-push: plain buffers from push_min_bytes(N), and every sharded
  // update (W' pushed, momentum sharded; see allreduce_push_kernel)
  {
    const bool shard_ok = mode_sharded && (update_len & 3) == 0;
    const bool want = shard_ok ? (auto_route || req == MD_ROUTE_PUSH)
                               : epi == 0 && (req == MD_ROUTE_PUSH ||
                                              (auto_route && n * 4 >= push_min_bytes(N)));
    if (want && fold_ok && avail >= 1) {
      // tile: deep enough rings for the N sources (measured, graph-timed 1 GiB:
      // N = 4 2048 -> 2361 us vs 4096 -> 2596 us; N = 2 3072 -> 1615 vs 1636)
      int64_t TE = tile_req ? tile_req : (N == 2 ? 3072 : 2048);
      int64_t A0, B0;
      push_slice(n, N, 0, &A0, &B0);
      if (!tile_req) {  // balanced: every CTA gets the same number of tiles (no ragged last wave)
        const int64_t rounds = std::max<int64_t>(1, (B0 - A0 + avail * TE - 1) / (avail * TE));
        TE = std::max<int64_t>(4, ((B0 - A0 + avail * rounds - 1) / (avail * rounds) + 3) &
                                      ~int64_t(3));
      }
      while ((B0 - A0 + TE - 1) / TE > kMaxTiles) TE *= 2;
      const int ups = epi == 0 ? 0 : (epi >= 3 ? 2 : 1);
      const int64_t stage_bytes = static_cast<int64_t>(N + 1 + ups) * TE * 4;
      // ring: the 192 KB of round 1 for plain calls (measured: a 6th stage from
      // the 224 KB ring made 1 GiB at N = 2 3 % slower), 224 KB when the W /
      // momentum rows ride along (sharded update)
      const int64_t ring = epi == 0 ? kRingBytes : kStreamRingBytes;
      const int S = static_cast<int>(std::min<int64_t>(8, ring / stage_bytes));
      if (S >= 2) {
        const int64_t T = std::max<int64_t>(1, (B0 - A0 + TE - 1) / TE);
        const int g = static_cast<int>(std::min<int64_t>(avail, T));
        a.seg = TE;
        a.lag = S;
        a.ctas_per_view = g;
        a.sharded = shard_ok;
        a.exit_sys_release = 1;
        a.cfg_word = cfg_word_of(MD_ROUTE_PUSH, false, shard_ok, TE);
        const void* k = allreduce_push_kernel_of(epi);
        const size_t smem = static_cast<size_t>(S) * stage_bytes;
        int rc = smem_attr_once(k, dev, kStreamRingBytes);
        if (rc == MD_OK) rc = setup_trace(&a, dev, g, n_views);
        if (rc == MD_OK) rc = launch_views(k, g, n_views, smem, &a, stream);
        if (rc == MD_OK) record_route(dev, MD_ROUTE_PUSH, TE, shard_ok);
        return rc;
      }
    }
  }

  // ---- LL push (the smallest buffers): see allreduce_ll_kernel
  {
    const int64_t g0 = std::min<int64_t>(avail, std::max<int64_t>(1, (n + 255) / 256));
    const int64_t E = g0 > 0 ? (((n + g0 - 1) / g0) + 3) & ~int64_t(3) : 0;
    const bool want = req == MD_ROUTE_LL || (auto_route && n * 4 <= ll_max_bytes(N));
    if (want && fold_ok && n <= kLLElems && avail >= 1 && N * E * 4 <= int64_t(kRingBytes)) {
      const int64_t g = (n + E - 1) / E;
      a.seg = E;
      a.ctas_per_view = static_cast<int32_t>(g);
      const void* k = allreduce_ll_kernel_of(epi);
      int rc = smem_attr_once(k, dev, kRingBytes);
      if (rc == MD_OK)
        rc = launch_views(k, static_cast<unsigned>(g), n_views, static_cast<size_t>(N) * E * 4,
                          &a, stream);
      if (rc == MD_OK) record_route(dev, MD_ROUTE_LL, E, false);
      return rc;
    }
  }

  // ---- one-shot pull (buffers that fit one SMEM pass of every rank's data)
  {
    const int64_t emax = static_cast<int64_t>(kRingBytes / 4u / N) & ~int64_t(3);
    int64_t g = std::min<int64_t>(avail, std::max<int64_t>(1, (n + 1023) / 1024));
    const int64_t E = (((n + g - 1) / g) + 3) & ~int64_t(3);
    const bool want = req == MD_ROUTE_ONESHOT || (auto_route && n * 4 <= oneshot_max_bytes(N));
    if (want && fold_ok && avail >= 1 && E <= emax) {
      g = (n + E - 1) / E;
      a.seg = E;
      a.ctas_per_view = static_cast<int32_t>(g);
      a.cfg_word = cfg_word_of(MD_ROUTE_ONESHOT, false, false, E);
      const void* k = allreduce_oneshot_kernel_of(epi);
      int rc = smem_attr_once(k, dev, kRingBytes);
      if (rc == MD_OK)
        rc = launch_views(k, static_cast<unsigned>(g), n_views, static_cast<size_t>(N) * E * 4,
                          &a, stream);
      if (rc == MD_OK) record_route(dev, MD_ROUTE_ONESHOT, E, false);
      return rc;
    }
  }

  // ---- stream (all-pull, tiled): replicated fused calls at N = 2 from 64 MiB,
  // balanced tiles of <= 6656 floats (two stages of [2 ranks | W | momentum]
  // in the 224 KB ring): C5 step at N = 2, graph-timed, 206 -> 198 us
  // (profiles/README.md). At N > 2 it pulls (N-1) x bytes and loses (N = 4:
  // 502 vs 275 us), so there it only runs when asked for.
  {
    const bool want =
        req == MD_ROUTE_STREAM || (auto_route && N == 2 && epi != 0 && n * 4 >= kStreamMinBytes);
    if (want && fold_ok && avail >= 1) {
      int64_t TE = 2048;
      if (N == 2) {  // balanced: every CTA gets the same number of tiles
        const int64_t rounds = std::max<int64_t>(1, (n + avail * 6656 - 1) / (avail * 6656));
        TE = std::max<int64_t>(4, ((n + avail * rounds - 1) / (avail * rounds) + 3) & ~int64_t(3));
      }
      if (tile_req) TE = tile_req;
      while ((n + TE - 1) / TE > kMaxTiles) TE *= 2;
      const int epi_slots = epi == 0 ? 0 : (epi >= 3 ? 2 : 1);
      const int64_t stage_bytes = static_cast<int64_t>(N + epi_slots) * TE * 4;
      const int S = static_cast<int>(std::min<int64_t>(8, kStreamRingBytes / stage_bytes));
      if (S >= 2) {
        const int64_t T = (n + TE - 1) / TE;
        const int g = static_cast<int>(std::min<int64_t>(avail, T));
        a.seg = TE;
        a.lag = S;
        a.ctas_per_view = g;
        a.cfg_word = cfg_word_of(MD_ROUTE_STREAM, false, false, TE);
        const void* k = allreduce_stream_kernel_of(epi);
        int rc = smem_attr_once(k, dev, kStreamRingBytes);
        if (rc == MD_OK)
          rc = launch_views(k, g, n_views, static_cast<size_t>(S) * stage_bytes, &a, stream);
        if (rc == MD_OK) record_route(dev, MD_ROUTE_STREAM, TE, false);
        return rc;
      }
    }
  }

  // ---- the pipelined tree: every other call (fused updates at N > 2, worker
  // folds, unaligned buffers). The owner-computes schedule
  // (md_plan_set_schedule, build_owner_plans) runs the same channelized
  // kernel over the owner plan (n slices), each owner evaluating the plan's
  // fold programs; worker folds and unaligned buffers keep the tree schedule
  // (same bits either way).
  auto weighted_of = [&](const std::vector<RankPlan>& plans) {
    int wmax = 0;
    for (const RankPlan& rp : plans) {
      int wt = 0;
      for (int i = 0; i < rp.n_tasks; ++i) {
        const Task& t = rp.t[i];
        wt += t.type == 1 || t.n_fold > 1 || t.parent < 0 || n_workers > 0;
      }
      wmax = std::max(wmax, wt);
    }
    return wmax;
  };
  // (the owner plan needs the channelized kernel: one CTA per task at least)
  const bool owner = plan->schedule == MD_SCHED_OWNER && N > 1 && n_workers == 0 && a.vec_ok &&
                     req != MD_ROUTE_QUEUE && plan->owner_dev && plan->prog_dev &&
                     weighted_of(plan->owner_host) <= avail;
  const std::vector<RankPlan>& hp = owner ? plan->owner_host : plan->host;
  if (owner) {
    a.plan = plan->owner_dev;
    a.k = N;
    const int64_t ml = (n + N - 1) / N;
    const int64_t sg =
        std::min(std::max<int64_t>(4, (seg_elems + 3) & ~int64_t(3)), auto_seg(ml, dev));
    const int64_t ms = ((ml + 3) / kMaxSegs + 4 + 3) & ~int64_t(3);
    a.seg = std::max(sg, ms);
    int64_t mx2 = 0;
    for (int col = 0; col < N; ++col) {
      int64_t st, ln;
      chunk_of(n, N, col, &st, &ln);
      mx2 = std::max(mx2, nseg_of(st, ln, a.seg));
    }
    a.max_nseg = static_cast<int32_t>(mx2);
  }
  // 16-byte aligned buffers take the channelized TMA kernel; anything else
  // the work-queue kernel with its scalar path (MD_ROUTE_QUEUE forces it)
  // (and only when every task of every rank can own at least one CTA)
  const bool chan = a.vec_ok && req != MD_ROUTE_QUEUE && weighted_of(hp) <= avail;
  const void* kern = chan ? allreduce_channels_kernel_of(epi) : allreduce_kernel_of(epi);
  int rc = smem_attr_once(kern, dev, kRingBytes);
  if (rc != MD_OK) return rc;
  int per_sm = 0;
  MD_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kArThreads,
                                                             kRingBytes));
  const int resident = per_sm * sm_count(dev);
  if (ctas <= 0) ctas = resident / n_views;
  ctas = std::min(ctas, resident / n_views);
  if (ctas < 1) {
    set_error("%d views do not fit co-resident on device %d", n_views, dev);
    return MD_ERR_INVALID_CONFIG;
  }
  a.ctas_per_view = ctas;
  // lag: about one CTA wave of items per pipeline stage (override: MD_AR_LAG)
  int max_stage = 0, max_tasks = 1;
  for (const RankPlan& rp : hp) {
    max_tasks = std::max(max_tasks, rp.n_tasks);
    for (int i = 0; i < rp.n_tasks; ++i) max_stage = std::max(max_stage, rp.t[i].stage);
  }
  a.lag = env.lag >= 0 ? env.lag : std::max(1, ctas / max_tasks);
  a.max_stage = max_stage;
  // the queue and channelized kernels exchange the same per-segment flags
  a.cfg_word = cfg_word_of(MD_ROUTE_TREE, owner, false, a.seg);
  rc = setup_trace(&a, dev, ctas, n_views);
  if (rc == MD_OK) rc = launch_views(kern, ctas, n_views, kRingBytes, &a, stream);
  if (rc == MD_OK) record_route(dev, chan ? MD_ROUTE_TREE : MD_ROUTE_QUEUE, a.seg, false);
  return rc;
}

}  // extern "C"

extern "C" int md_trace_dump(int32_t device, const char* path) {
  if (device < 0 || device >= 64 || !g_trace[device].ptr) {
    set_error("no allreduce trace on device %d (set MD_AR_TRACE=1)", device);
    return MD_ERR_INVALID_CONFIG;
  }
  std::vector<char> host(g_trace[device].used);
  int prev;
  MD_CUDA_TRY(cudaGetDevice(&prev));
  MD_CUDA_TRY(cudaSetDevice(device));
  cudaError_t e = cudaMemcpy(host.data(), g_trace[device].ptr, host.size(), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemset(g_trace[device].ptr, 0, g_trace[device].bytes);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    set_error("trace copy: %s", cudaGetErrorString(e));
    return MD_ERR_CUDA;
  }
  FILE* f = fopen(path, "wb");
  if (!f) {
    set_error("cannot write %s", path);
    return MD_ERR_INVALID_CONFIG;
  }
  fwrite(host.data(), 1, host.size(), f);
  fclose(f);
  return MD_OK;
}
