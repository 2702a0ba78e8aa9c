// Internal definitions shared by the allreduce translation units of
// libmdb200 (sm_100a): the peer-mapped control block, fold plans and fold
// programs, the kernel argument block, and the device helpers every route
// uses (chunk geometry, fold programs, flag waits, the SGD epilogue, the
// entry / exit barriers). The kernels live in md_ar_tree.cu (pipelined tree,
// work queue), md_ar_direct.cu (LL push, one-shot pull, stream) and
// md_ar_push.cu (owner-push); md_allreduce.cu holds the host side (plans,
// communicators, the route dispatcher).
//
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
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "md_common.cuh"

namespace md {

constexpr int kMaxSegs = 4096;        // per color
constexpr int kLLElems = 262144;      // LL inbox: payload floats per (parity, source)
constexpr int kMaxTiles = 65536;      // stream kernel: tiles per call
constexpr int kArThreads = 512;
constexpr int kChanThreads = 384;  // channelized tree kernel (see md_ar_tree.cu)
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
static __device__ bool wait_flag(const ViewArgs& v, const uint32_t* flag, uint32_t epoch,
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
static __device__ bool entry_barrier(const AllreduceArgs& a, const ViewArgs& v, int local_cta,
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
static __device__ void exit_barrier(const AllreduceArgs& a, const ViewArgs& v, uint32_t epoch) {
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

__device__ __forceinline__ bool aborted(const ViewArgs& v) {
  return *reinterpret_cast<volatile uint32_t*>(&v.ctrl->abort_flag) != 0;
}

// 16-byte aligned owner slice j of an n-element buffer (owner-push; the tail
// n & 3 is not in any slice)
__host__ __device__ __forceinline__ void push_slice(int64_t n, int N, int j, int64_t* lo,
                                                    int64_t* hi) {
  const int64_t n4 = n & ~int64_t(3);
  const int64_t per = ((n4 / 4 + N - 1) / N) * 4;
  const int64_t l = static_cast<int64_t>(j) * per, h = static_cast<int64_t>(j + 1) * per;
  *lo = l < n4 ? l : n4;
  *hi = h < n4 ? h : n4;
}


// kernel of each route for an epilogue variant (0 none, 1 SGD, 2 + wd,
// 3 + momentum, 4 momentum + wd), defined next to the kernels
const void* allreduce_kernel_of(int epi);
const void* allreduce_channels_kernel_of(int epi);
const void* allreduce_ll_kernel_of(int epi);
const void* allreduce_oneshot_kernel_of(int epi);
const void* allreduce_stream_kernel_of(int epi);
const void* allreduce_push_kernel_of(int epi);

#define MD_EPI_TABLE(kernel)                                                                   \
  const void* kernel##_of(int epi) {                                                           \
    switch (epi) {                                                                             \
      case 1: return reinterpret_cast<const void*>(kernel<1>);                                 \
      case 2: return reinterpret_cast<const void*>(kernel<2>);                                 \
      case 3: return reinterpret_cast<const void*>(kernel<3>);                                 \
      case 4: return reinterpret_cast<const void*>(kernel<4>);                                 \
      default: return reinterpret_cast<const void*>(kernel<0>);                                \
    }                                                                                          \
  }

}  // namespace md
