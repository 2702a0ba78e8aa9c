// Allreduce routes that evaluate each color's fold program locally on data
// moved in one pass (sm_100a): the LL push kernel (smallest buffers), the
// one-shot pull kernel and the tiled all-pull stream kernel. Same adds in the
// same order as the color trees (ColorProg), so the same bits.
#include "md_allreduce.cuh"

namespace md {

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


MD_EPI_TABLE(allreduce_ll_kernel)
MD_EPI_TABLE(allreduce_oneshot_kernel)
MD_EPI_TABLE(allreduce_stream_kernel)

}  // namespace md
