// Pipelined multi-color tree allreduce (sm_100a): the work-queue kernel
// (any alignment, scalar path) and the channelized kernel (TMA ring,
// warp-specialised producer / notifier / fold warps). Every node folds its own
// value and its children's subtree sums in child-list order (ref
// collectives.py:271-286) and the root's result travels back down the tree
// (:289-296); the optional worker-fold prologue and SGD epilogue are fused.
#include "md_allreduce.cuh"

namespace md {

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
constexpr int kConsumerWarps = kChanThreads / 32 - 2;
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
__global__ void __launch_bounds__(kChanThreads, 1)
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


MD_EPI_TABLE(allreduce_kernel)
MD_EPI_TABLE(allreduce_channels_kernel)

}  // namespace md
