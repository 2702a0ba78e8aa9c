// Owner-push allreduce (sm_100a): plain calls and the sharded SGD update.
#include "md_allreduce.cuh"

namespace md {

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


MD_EPI_TABLE(allreduce_push_kernel)

}  // namespace md
