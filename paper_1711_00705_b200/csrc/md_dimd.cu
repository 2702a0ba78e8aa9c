// DIMD (distributed in-memory dataset) on B200: /root/reference/pkg/src/minidist/dimd.py
//
// Every random index is bit-exact with the reference, whose randomness is
// numpy's Generator(Philox(key)) (dimd.py:218, :309, :337-339):
//   * Philox4x64-10, counter pre-incremented, 32-bit draws take the low then
//     the high half of each 64-bit output (md_common.cuh);
//   * integers(0, n, size) = 32-bit Lemire with rejection per draw;
//   * permutation(n) = Fisher-Yates over arange(n), i = n-1 .. 1, with
//     j = random_interval(i) (masked rejection).
//
// The shuffle (Algorithm 2, dimd.py:281-350) is restructured for NVLink:
// each receiving rank recomputes every group member's destination draws (one
// Philox word per record -- cheap), so it knows, before any byte moves, the
// receive order (segment, source member, source order), its record count N'
// and its final permutation. Fisher-Yates is reconstructed in parallel: the
// sequential part is reduced to picking which 32-bit words are accepted
// (one warp), then "who ends where" follows from a stable radix sort of the
// swap targets plus pointer jumping. The segmented alltoallv
// becomes ONE pull kernel: every output record is read straight from its
// source member's blob through peer memory into its final slot.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>

#include "md_common.cuh"

namespace md {

constexpr uint64_t kRoleDest = 0x74736564ULL;  // int.from_bytes(b"dest", "little")
constexpr uint64_t kRolePerm = 0x6d726570ULL;  // b"perm"

// ---- bounded integers (numpy random_bounded_uint64_fill, 32-bit Lemire) ------
// Value of draw k assuming no earlier rejection in the stream. Returns false
// when the draw itself would be rejected (caller falls back to a serial pass).
__device__ __forceinline__ bool lemire_fast(uint64_t key, uint64_t k, uint32_t S, uint32_t* out) {
  uint64_t m = static_cast<uint64_t>(philox_word32(key, k)) * S;
  uint32_t left = static_cast<uint32_t>(m);
  if (left < S) {
    uint32_t thr = static_cast<uint32_t>((0x100000000ULL - S) % S);
    if (left < thr) return false;
  }
  *out = static_cast<uint32_t>(m >> 32);
  return true;
}

// Serial exact draws [0, count) of integers(0, S) (S >= 2).
__device__ void lemire_serial(uint64_t key, uint64_t count, uint32_t S, int32_t* out32,
                              int64_t* out64) {
  uint64_t w = 0;
  uint32_t thr = static_cast<uint32_t>((0x100000000ULL - S) % S);
  for (uint64_t k = 0; k < count; ++k) {
    uint64_t m = static_cast<uint64_t>(philox_word32(key, w++)) * S;
    if (static_cast<uint32_t>(m) < S) {
      while (static_cast<uint32_t>(m) < thr) m = static_cast<uint64_t>(philox_word32(key, w++)) * S;
    }
    uint32_t v = static_cast<uint32_t>(m >> 32);
    if (out32) out32[k] = static_cast<int32_t>(v);
    if (out64) out64[k] = static_cast<int64_t>(v);
  }
}

// The same stream, block-parallel: numpy's Lemire-with-rejection makes draw k
// the k-th Philox word w (w = 0, 1, ...) whose low product half is >= thr
// (a first try with left < S re-tests left < thr, so "rejected" is exactly
// left < thr). One CTA (blockDim % 32 == 0, every thread calls) compacts the
// accepted words tile by tile with a ballot prefix. S >= 2.
__device__ void block_lemire_compact(uint64_t key, uint32_t S, int64_t count, int64_t* out) {
  __shared__ int warp_tot[32];
  __shared__ long long s_have;
  const uint32_t thr = static_cast<uint32_t>((0x100000000ULL - S) % S);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  if (tid == 0) s_have = 0;
  __syncthreads();
  for (uint64_t base = 0;; base += blockDim.x) {
    const long long have = s_have;
    if (have >= count) break;
    const uint64_t m = static_cast<uint64_t>(philox_word32(key, base + tid)) * S;
    const bool acc = static_cast<uint32_t>(m) >= thr;
    const unsigned bal = __ballot_sync(0xffffffffu, acc);
    if (lane == 0) warp_tot[wid] = __popc(bal);
    __syncthreads();
    int off = __popc(bal & ((1u << lane) - 1u));
    for (int w = 0; w < wid; ++w) off += warp_tot[w];
    if (acc && have + off < count) out[have + off] = static_cast<int64_t>(m >> 32);
    __syncthreads();
    if (tid == 0) {
      int t = 0;
      for (int w = 0; w < nw; ++w) t += warp_tot[w];
      s_have = have + t;
    }
    __syncthreads();
  }
}

// random_batch picks (n_records may exceed 2^32 only in theory; the 32-bit
// path covers n <= 2^32 exactly as numpy does).
__global__ void picks_kernel(uint64_t key, uint32_t n, int64_t batch, int64_t* picks, int* bad) {
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= batch) return;
  if (n == 1) {
    picks[i] = 0;
    return;
  }
  uint32_t v;
  if (lemire_fast(key, static_cast<uint64_t>(i), n, &v)) picks[i] = v;
  else atomicExch(bad, 1);
}
__global__ void __launch_bounds__(1024) picks_block_kernel(uint64_t key, uint32_t n,
                                                           int64_t batch, int64_t* picks) {
  const int i = threadIdx.x;
  int rejected = 0;
  if (i < batch) {
    uint32_t v = 0;
    if (n == 1) picks[i] = 0;
    else if (lemire_fast(key, static_cast<uint64_t>(i), n, &v)) picks[i] = v;
    else rejected = 1;
  }
  if (__syncthreads_or(rejected))  // rare: redo the stream with the rejections
    block_lemire_compact(key, n, batch, picks);
}
// Graph-replayable variant: key from a device step counter, which it advances.
__global__ void __launch_bounds__(1024) picks_step_kernel(uint64_t seed, uint64_t role,
                                                          uint64_t worker, int64_t* step,
                                                          uint32_t n, int64_t batch,
                                                          int64_t* picks) {
  const int64_t st = *step;
  const uint64_t key =
      mix64_step(mix64_step(mix64_step(mix64_step(0, seed), role), worker),
                 static_cast<uint64_t>(st));
  const int i = threadIdx.x;
  int rejected = 0;
  if (i < batch) {
    uint32_t v = 0;
    if (n == 1) picks[i] = 0;
    else if (lemire_fast(key, static_cast<uint64_t>(i), n, &v)) picks[i] = v;
    else rejected = 1;
  }
  if (__syncthreads_or(rejected)) block_lemire_compact(key, n, batch, picks);
  if (i == 0) *step = st + 1;  // every thread read *step before the barrier above
}
__global__ void __launch_bounds__(1024) picks_fix_kernel(uint64_t key, uint32_t n,
                                                         int64_t batch, int64_t* picks,
                                                         const int* bad) {
  if (*bad) block_lemire_compact(key, n, batch, picks);
}

// ---- shuffle: destination draws of every source member ----------------------
struct SrcTable {
  int64_t n_rec[MD_MAX_GROUP];
  int64_t base[MD_MAX_GROUP + 1];  // prefix of n_rec
};

__host__ __device__ __forceinline__ int64_t seg_lo(int64_t t, int64_t n, int64_t m) {
  return t * n / m;  // dimd.py:304
}

__device__ __forceinline__ int64_t seg_of(int64_t i, int64_t n, int64_t m) {
  int64_t t = (i * m) / (n > 0 ? n : 1);
  if (t >= m) t = m - 1;
  while (t + 1 < m && seg_lo(t + 1, n, m) <= i) ++t;
  while (t > 0 && seg_lo(t, n, m) > i) --t;
  return t;
}

__device__ __forceinline__ uint64_t dest_key(uint64_t seed, uint64_t group, uint64_t q, uint64_t t) {
  uint64_t acc = 0;
  acc = mix64_step(acc, seed);
  acc = mix64_step(acc, kRoleDest);
  acc = mix64_step(acc, group);
  acc = mix64_step(acc, q);
  acc = mix64_step(acc, t);
  return acc;
}

__global__ void dest_kernel(const __grid_constant__ SrcTable tab, int32_t S, int64_t m,
                            uint64_t seed, uint64_t group, int64_t total, int32_t* dest,
                            uint8_t* seg_bad) {
  int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= total) return;
  int q = 0;
  while (tab.base[q + 1] <= g) ++q;
  int64_t i = g - tab.base[q];
  int64_t n = tab.n_rec[q];
  if (S == 1) {
    dest[g] = 0;
    return;
  }
  int64_t t = seg_of(i, n, m);
  uint32_t v;
  if (lemire_fast(dest_key(seed, group, q, t), static_cast<uint64_t>(i - seg_lo(t, n, m)),
                  static_cast<uint32_t>(S), &v))
    dest[g] = static_cast<int32_t>(v);
  else
    seg_bad[q * m + t] = 1;
}

// serial redo of the (q, t) segments that hit a Lemire rejection
__global__ void dest_fix_kernel(const __grid_constant__ SrcTable tab, int32_t S, int64_t m,
                                uint64_t seed, uint64_t group, int32_t* dest,
                                const uint8_t* seg_bad) {
  int64_t qt = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (qt >= S * m) return;
  if (!seg_bad[qt]) return;
  int q = static_cast<int>(qt / m);
  int64_t t = qt % m, n = tab.n_rec[q];
  int64_t lo = seg_lo(t, n, m), hi = seg_lo(t + 1, n, m);
  lemire_serial(dest_key(seed, group, q, t), static_cast<uint64_t>(hi - lo),
                static_cast<uint32_t>(S), dest + tab.base[q] + lo, nullptr);
}

__global__ void mine_flag_kernel(const int32_t* dest, int64_t total, int32_t me, int32_t* flag) {
  int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g < total) flag[g] = dest[g] == me;
}

// records per destination member: every member's record count after this
// shuffle (the next shuffle's n_rec, so it can start its plan before the
// counts' host collective returns)
__global__ void dest_count_kernel(const int32_t* dest, int64_t total, int32_t S,
                                  unsigned long long* cnt) {
  __shared__ unsigned int h[MD_MAX_GROUP];
  for (int q = threadIdx.x; q < S; q += blockDim.x) h[q] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    atomicAdd(&h[dest[i]], 1u);
  __syncthreads();
  for (int q = threadIdx.x; q < S; q += blockDim.x)
    if (h[q]) atomicAdd(&cnt[q], static_cast<unsigned long long>(h[q]));
}

// receive-order bases: base[t][q] in (t-major, q) order -- dimd.py:303-335
__global__ void recv_base_kernel(const __grid_constant__ SrcTable tab, int32_t S, int64_t m,
                                 const int32_t* excl /* total+1 entries */, int64_t* base_tq,
                                 int64_t* n_final) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  int64_t acc = 0;
  for (int64_t t = 0; t < m; ++t) {
    for (int q = 0; q < S; ++q) {
      int64_t n = tab.n_rec[q];
      int64_t lo = tab.base[q] + seg_lo(t, n, m), hi = tab.base[q] + seg_lo(t + 1, n, m);
      base_tq[t * S + q] = acc;
      acc += static_cast<int64_t>(excl[hi]) - excl[lo];
    }
  }
  *n_final = acc;
}

__global__ void got_scatter_kernel(const __grid_constant__ SrcTable tab, int32_t S, int64_t m,
                                   int64_t total, const int32_t* flag, const int32_t* excl,
                                   const int64_t* base_tq, int32_t* got_member, int64_t* got_rec) {
  int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g >= total || !flag[g]) return;
  int q = 0;
  while (tab.base[q + 1] <= g) ++q;
  int64_t i = g - tab.base[q], n = tab.n_rec[q];
  int64_t t = seg_of(i, n, m);
  int64_t lo = tab.base[q] + seg_lo(t, n, m);
  int64_t G = base_tq[t * S + q] + (excl[g] - excl[lo]);
  got_member[G] = q;
  got_rec[G] = i;
}

// ---- permutation(N') ------------------------------------------------------------
__global__ void words_kernel(uint64_t key, int64_t first_word, int64_t count, uint32_t* ws) {
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < count) ws[i] = philox_word32(key, static_cast<uint64_t>(first_word + i));
}

__device__ __forceinline__ uint32_t mask_of(uint32_t s) {
  uint32_t m = s;
  m |= m >> 1;
  m |= m >> 2;
  m |= m >> 4;
  m |= m >> 8;
  m |= m >> 16;
  return m;
}

// One warp: walk the word stream deciding which word each Fisher-Yates step
// accepts (random_interval: v = word & mask(s), accepted iff v <= s).
// state[0] = next step s (counts down), state[1] = next word index;
// resumable when it runs out of pre-generated words.
//
// 64 words per step of the walk (two per lane). With the same mask for steps
// s .. s-63 a word is accepted for sure if v <= s-63 and rejected for sure if
// v > s; only words in between ("ambiguous") depend on how many earlier words
// were accepted. So: consume every word up to and including the FIRST
// ambiguous one -- the ones before it are decided, and it is decided exactly
// by the count of accepted words before it. Words reach SMEM in 32 KiB tiles
// by one TMA bulk copy each. (The serial one-word-at-a-time walk is left only
// for s < 128 and windows where the mask changes.)
constexpr int kFyTile = 8192;
__global__ void __launch_bounds__(32) fy_scan_kernel(const uint32_t* ws, int64_t n_words,
                                                     int64_t word_base, uint32_t* J,
                                                     int64_t* state) {
  __shared__ __align__(128) uint32_t tile[kFyTile];
  __shared__ __align__(8) uint64_t bar;
  constexpr uint32_t kAll = 0xffffffffu;
  const int lane = threadIdx.x;
  const uint32_t lt = (1u << lane) - 1u;
  int64_t s = state[0];
  int64_t p = state[1];
  int64_t t_lo = 0, t_hi = 0;  // tile = words [t_lo, t_hi) relative to word_base
  uint32_t phase = 0;
  if (lane == 0) {
    mbar_init(&bar, 1);
    mbar_init_fence();
  }
  __syncwarp();
  uint32_t mask = mask_of(static_cast<uint32_t>(s));
  while (s > 0) {
    const int64_t rel = p - word_base;
    if (rel + 64 + 3 > n_words) break;  // need more words (host resumes at p)
    if (rel + 64 > t_hi) {
      const int64_t lo = rel & ~int64_t(3);  // 16-byte aligned source
      const int64_t cnt = min(static_cast<int64_t>(kFyTile), (n_words - lo) & ~int64_t(3));
      __syncwarp();
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar, static_cast<uint32_t>(cnt * 4));
        tma_load_1d(tile, ws + lo, static_cast<uint32_t>(cnt * 4), &bar);
      }
      while (!mbar_try_wait(&bar, phase)) {
      }
      phase ^= 1;
      t_lo = lo;
      t_hi = lo + cnt;
    }
    const int base = static_cast<int>(rel - t_lo);
    if (s >= 128 && mask_of(static_cast<uint32_t>(s - 63)) == mask) {
      const uint32_t su = static_cast<uint32_t>(s), sure = su - 63;
      const uint32_t v0 = tile[base + lane] & mask, v1 = tile[base + 32 + lane] & mask;
      const bool a0 = v0 <= sure, a1 = v1 <= sure;
      const uint32_t A0 = __ballot_sync(kAll, a0), A1 = __ballot_sync(kAll, a1);
      const uint32_t M0 = __ballot_sync(kAll, !a0 && v0 <= su);
      const uint32_t M1 = __ballot_sync(kAll, !a1 && v1 <= su);
      uint32_t acc0 = A0, acc1 = A1;
      int used = 64;
      if (M0) {
        const int f = __ffs(M0) - 1;
        acc0 = A0 & ((1u << f) - 1u);
        acc1 = 0;
        if (__shfl_sync(kAll, v0, f) <= su - __popc(acc0)) acc0 |= 1u << f;
        used = f + 1;
      } else if (M1) {
        const int f = __ffs(M1) - 1;
        acc1 = A1 & ((1u << f) - 1u);
        if (__shfl_sync(kAll, v1, f) <= su - __popc(acc0) - __popc(acc1)) acc1 |= 1u << f;
        used = 33 + f;
      }
      const int c0 = __popc(acc0);
      if ((acc0 >> lane) & 1u) J[s - __popc(acc0 & lt)] = v0;
      if ((acc1 >> lane) & 1u) J[s - c0 - __popc(acc1 & lt)] = v1;
      s -= c0 + __popc(acc1);
      mask = mask_of(static_cast<uint32_t>(s));
      p += used;
      continue;
    }
    const uint32_t my = tile[base + lane];
    int used = 32;
    for (int l = 0; l < 32; ++l) {
      uint32_t v = __shfl_sync(kAll, my, l) & mask;
      if (v <= static_cast<uint32_t>(s)) {
        if (lane == 0) J[s] = v;
        --s;
        mask = mask_of(static_cast<uint32_t>(s));
        if (s == 0) {
          used = l + 1;
          break;
        }
      }
    }
    p += used;
  }
  if (lane == 0) {
    state[0] = s;
    state[1] = p;
  }
}

__global__ void iota_kernel(uint32_t* v, int64_t n, uint32_t first) {
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) v[i] = first + static_cast<uint32_t>(i);
}

__global__ void fill_i32_kernel(int32_t* v, int64_t n, int32_t x) {
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) v[i] = x;
}

// sorted (target, step) pairs -> nxt[step] (next later step with the same
// target) and parent[q] (first step > q whose target is q)
__global__ void fy_links_kernel(const uint32_t* tgt, const uint32_t* stp, int64_t m_pairs,
                                int32_t* nxt, int32_t* parent) {
  int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (p >= m_pairs) return;
  uint32_t q = tgt[p], s = stp[p];
  bool has_next = p + 1 < m_pairs && tgt[p + 1] == q;
  if (has_next) nxt[s] = static_cast<int32_t>(stp[p + 1]);
  bool first = p == 0 || tgt[p - 1] != q;
  if (first) {
    if (s != q) parent[q] = static_cast<int32_t>(s);
    else if (has_next) parent[q] = static_cast<int32_t>(stp[p + 1]);
  }
}

__global__ void ptr_init_kernel(const int32_t* parent, int64_t n, int32_t* ptr) {
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) ptr[i] = parent[i] >= 0 ? parent[i] : static_cast<int32_t>(i);
}
__global__ void ptr_jump_kernel(const int32_t* in, int64_t n, int32_t* out, int* changed) {
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  int32_t a = in[i], b = in[a];
  out[i] = b;
  if (b != a) *changed = 1;
}

// a[s] (s >= 1) and a[0]; then final = got[a]
__global__ void fy_final_kernel(const int32_t* nxt, const int32_t* root, const uint32_t* J,
                                const uint32_t* tgt, const uint32_t* stp, int64_t n,
                                const int32_t* got_member, const int64_t* got_rec,
                                int32_t* final_member, int64_t* final_rec) {
  int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (s >= n) return;
  int64_t a;
  if (s == 0) {
    a = (n > 1 && tgt[0] == 0) ? root[stp[0]] : 0;
  } else {
    int32_t w = nxt[s];
    a = w >= 0 ? root[w] : static_cast<int64_t>(J[s]);
  }
  final_member[s] = got_member[a];
  final_rec[s] = got_rec[a];
}

// ---- index rebuild + record movement --------------------------------------------
struct PeerIdx {
  const uint32_t* len[MD_MAX_GROUP];
  const uint32_t* label[MD_MAX_GROUP];
};
struct PeerBlob {
  const uint8_t* blob[MD_MAX_GROUP];
  const uint64_t* off[MD_MAX_GROUP];
};

__global__ void index_kernel(const __grid_constant__ PeerIdx p, const int32_t* fm,
                             const int64_t* fr, int64_t n, uint32_t* out_len, uint32_t* out_label,
                             unsigned long long* len64) {
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  int q = fm[i];
  int64_t r = fr[i];
  uint32_t L = p.len[q][r];
  out_len[i] = L;
  out_label[i] = p.label[q][r];
  len64[i] = L;
}

// Copy `len` bytes src -> dst with the whole CTA (16-byte vectors when the
// two addresses share their alignment mod 16).
__device__ __forceinline__ void cta_copy(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                         uint64_t len) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  uintptr_t sa = reinterpret_cast<uintptr_t>(src), da = reinterpret_cast<uintptr_t>(dst);
  if ((sa & 15) == (da & 15)) {
    uint64_t head = (16 - (sa & 15)) & 15;
    if (head > len) head = len;
    if (static_cast<uint64_t>(tid) < head) dst[tid] = src[tid];
    const uint4* s4 = reinterpret_cast<const uint4*>(src + head);
    uint4* d4 = reinterpret_cast<uint4*>(dst + head);
    uint64_t nv = (len - head) / 16;
    constexpr int U = 4;
    for (uint64_t b = tid; b < nv; b += static_cast<uint64_t>(nthr) * U) {
      uint4 x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        uint64_t k = b + static_cast<uint64_t>(u) * nthr;
        if (k < nv) x[u] = __ldcs(s4 + k);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        uint64_t k = b + static_cast<uint64_t>(u) * nthr;
        if (k < nv) __stcs(d4 + k, x[u]);
      }
    }
    uint64_t done = head + nv * 16;
    if (static_cast<uint64_t>(tid) < len - done) dst[done + tid] = src[done + tid];
  } else {
    for (uint64_t k = tid; k < len; k += nthr) dst[k] = src[k];
  }
}

__global__ void __launch_bounds__(512) pull_kernel(const __grid_constant__ PeerBlob p,
                                                   const int32_t* fm, const int64_t* fr,
                                                   int64_t n, const uint64_t* out_off,
                                                   const uint32_t* out_len, uint8_t* out) {
  for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
    int q = fm[i];
    int64_t r = fr[i];
    cta_copy(out + out_off[i], p.blob[q] + p.off[q][r], out_len[i]);
  }
}

// ---- push exchange (the bytes of dimd.py:303-335, sender side) -----------------
// The receiver groups its output slots by source member
// (md_shuffle_sendlist: a stable counting sort on final_member), so each
// source reads ONE contiguous list of (its record, output offset, length)
// per receiver and stores those records from its local blob straight into
// the receiver's new blob over NVLink (md_shuffle_push). Same placement as
// the pull, but the bytes cross the links as stores: measured bidirectional
// ceilings per GPU 681 GB/s for SM stores vs 625 GB/s for SM loads
// (profiles/r01_p2p_probe_n2.log), and no read-request traffic competes with
// the data in the other direction.
struct SendEntry {
  int64_t src_rec;   // record index in the source member's shard
  uint64_t dst_off;  // byte offset in the receiver's new blob
  uint32_t len;
  uint32_t pad;
};
static_assert(sizeof(SendEntry) == 24, "SendEntry is part of the peer-visible layout");

__global__ void member_count_kernel(const int32_t* fm, int64_t n, int32_t S,
                                    unsigned long long* cnt) {
  __shared__ unsigned int h[MD_MAX_GROUP];
  for (int q = threadIdx.x; q < S; q += blockDim.x) h[q] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    atomicAdd(&h[fm[i]], 1u);
  __syncthreads();
  for (int q = threadIdx.x; q < S; q += blockDim.x)
    if (h[q]) atomicAdd(&cnt[q], static_cast<unsigned long long>(h[q]));
}

__global__ void member_begin_kernel(const unsigned long long* cnt, int32_t S, int64_t* begin) {
  int64_t acc = 0;
  for (int q = 0; q < S; ++q) {
    begin[q] = acc;
    acc += static_cast<int64_t>(cnt[q]);
  }
  begin[S] = acc;
}

__global__ void sendlist_kernel(const int32_t* sorted_slot, const int32_t* fm, const int64_t* fr,
                                const uint64_t* out_off, const uint32_t* out_len, int64_t n,
                                SendEntry* list) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int32_t j = sorted_slot[i];
  SendEntry e;
  e.src_rec = fr[j];
  e.dst_off = out_off[j];
  e.len = out_len[j];
  e.pad = static_cast<uint32_t>(fm[j]);
  list[i] = e;
}

struct PushArgs {
  const SendEntry* list[MD_MAX_GROUP];  // receiver d's send list (peer-mapped)
  const int64_t* begin[MD_MAX_GROUP];   // receiver d's list offsets per source [S + 1]
  uint8_t* out[MD_MAX_GROUP];           // receiver d's new blob (peer-mapped)
};

// Work item i -> receiver (me + 1 + i mod S) mod S, entry i / S of our list
// there: every CTA wave spreads its stores over all receivers (a wave that
// targets one receiver would queue on that GPU's ingress). Thread 0 runs the
// items' metadata two steps ahead (the list entry of item i + 2G, the source
// offset of item i + G -- two dependent loads), so the chain's latency is off
// the copy's path, as in gather_kernel.
// kLocal: the one-member instance (S == 1, copies within the own HBM) is
// capped at 32 registers for 4 resident CTAs per SM (A/B: epoch 8.72 -> 8.39
// ms at N = 1); across GPUs the 64-register instance (2 CTAs per SM, the
// exchange grid) is faster (19.0 vs 19.3 ms at N = 2): the links, not the
// SM's loads in flight, bound it there.
template <bool kLocal>
__global__ void __launch_bounds__(512, kLocal ? 4 : 2) push_kernel(const __grid_constant__ PushArgs p, int32_t S,
                                                   int32_t me, const uint8_t* blob,
                                                   const uint64_t* off) {
  __shared__ int64_t lo[MD_MAX_GROUP], cnt[MD_MAX_GROUP];
  __shared__ int64_t s_items;
  __shared__ SendEntry s_e;
  __shared__ uint64_t s_src;
  __shared__ int s_ok;
  const int tid = threadIdx.x;
  if (tid < S) {
    const int64_t* b = p.begin[tid];
    lo[tid] = b[me];
    cnt[tid] = b[me + 1] - b[me];
  }
  __syncthreads();
  if (tid == 0) {
    int64_t mx = 0;
    for (int d = 0; d < S; ++d) mx = max(mx, cnt[d]);
    s_items = mx * S;
  }
  __syncthreads();
  const int64_t items = s_items;
  const int64_t G = gridDim.x;
  auto fetch = [&](int64_t i, SendEntry* en) -> bool {
    if (i >= items) return false;
    const int d = (me + 1 + static_cast<int>(i % S)) % S;
    const int64_t e = i / S;
    if (e >= cnt[d]) return false;
    *en = p.list[d][lo[d] + e];
    return true;
  };
  SendEntry e_cur{}, e_next{};
  uint64_t o_cur = 0;
  bool v_cur = false, v_next = false;
  if (tid == 0) {
    v_cur = fetch(blockIdx.x, &e_cur);
    o_cur = v_cur ? off[e_cur.src_rec] : 0;
    v_next = fetch(blockIdx.x + G, &e_next);
  }
  for (int64_t i = blockIdx.x; i < items; i += G) {
    if (tid == 0) {
      s_e = e_cur;
      s_src = o_cur;
      s_ok = v_cur;
      // advance the pipeline: offset of the next item, entry of the one after
      o_cur = v_next ? off[e_next.src_rec] : 0;
      e_cur = e_next;
      v_cur = v_next;
      v_next = fetch(i + 2 * G, &e_next);
    }
    __syncthreads();
    if (s_ok) {  // uniform across the CTA
      const int d = (me + 1 + static_cast<int>(i % S)) % S;
      const SendEntry en = s_e;
      cta_copy(p.out[d] + en.dst_off, blob + s_src, en.len);
    }
    __syncthreads();  // s_e / s_src are rewritten by the next item
  }
}

constexpr uint64_t kGatherChunk = 32 * 1024;

// kStep: the variant for training-step batches, which runs between the
// allreduce's 192-224 KB-SMEM kernels and therefore asks for the max-shared
// carveout (no L1/SMEM re-partition); bulk gathers take the other variant with
// the default carveout -- the max-shared one costs them 20 % (6.29 vs 5.03
// TB/s, tools/gather_variants.cu)
template <bool kStep>
__global__ void __launch_bounds__(512) gather_kernel(const uint8_t* blob, const uint64_t* off,
                                                     const uint32_t* len, const uint32_t* label,
                                                     const int64_t* picks, int64_t batch,
                                                     uint8_t* out, int64_t stride,
                                                     const uint64_t* out_off, uint32_t* out_label,
                                                     int32_t* bad, int chunks) {
  // work unit = (record, chunk of kGatherChunk bytes): a 32-record batch of
  // 150 KB images spreads over ~150 CTAs instead of 32. The next unit's
  // metadata (picks -> off/len, two dependent loads) is fetched while the
  // current chunk streams, so the chain's latency is off the copy's path.
  const int64_t units = batch * chunks;
  const int64_t G = gridDim.x;
  int64_t u = blockIdx.x;
  int64_t r = u < units ? picks[u / chunks] : 0;
  uint32_t L = u < units ? len[r] : 0;
  uint64_t o = u < units ? off[r] : 0;
  int64_t r_next = u + G < units ? picks[(u + G) / chunks] : 0;
  for (; u < units; u += G) {
    uint32_t L_next = 0;
    uint64_t o_next = 0;
    if (u + G < units) {
      L_next = len[r_next];
      o_next = off[r_next];
    }
    const int64_t r_after = u + 2 * G < units ? picks[(u + 2 * G) / chunks] : 0;
    const int64_t b = u / chunks;
    const int c = static_cast<int>(u % chunks);
    if (stride > 0 && static_cast<int64_t>(L) != stride) {
      if (threadIdx.x == 0 && bad && c == 0) atomicExch(bad, 1);
    } else {
      uint8_t* dst = stride > 0 ? out + b * stride : out + out_off[b];
      const uint64_t lo = chunks == 1 ? 0 : static_cast<uint64_t>(c) * kGatherChunk;
      if (lo < L) {
        const uint64_t n = chunks == 1 ? L : min(static_cast<uint64_t>(kGatherChunk), L - lo);
        cta_copy(dst + lo, blob + o + lo, n);
        if (threadIdx.x == 0 && c == 0 && out_label) out_label[b] = label[r];
      }
    }
    r = r_next;
    L = L_next;
    o = o_next;
    r_next = r_after;
  }
}


struct SegCopy {
  uint8_t* dst[MD_MAX_GROUP];
  const uint8_t* src[MD_MAX_GROUP];
  uint64_t len[MD_MAX_GROUP];
  uint64_t blocks_before[MD_MAX_GROUP + 1];  // CTA ranges per segment
};

// each segment gets a contiguous range of CTAs proportional to its size;
// every CTA copies a 256 KiB slice of it
constexpr uint64_t kSliceBytes = 256 * 1024;
__global__ void __launch_bounds__(512) segcopy_kernel(const __grid_constant__ SegCopy p, int n) {
  int seg = 0;
  while (seg + 1 <= n && p.blocks_before[seg + 1] <= blockIdx.x) ++seg;
  if (seg >= n) return;
  uint64_t slice = blockIdx.x - p.blocks_before[seg];
  uint64_t lo = slice * kSliceBytes;
  if (lo >= p.len[seg]) return;
  uint64_t L = p.len[seg] - lo < kSliceBytes ? p.len[seg] - lo : kSliceBytes;
  cta_copy(p.dst[seg] + lo, p.src[seg] + lo, L);
}

// ---- synthetic corpus -------------------------------------------------------------
__device__ __forceinline__ uint32_t synth_word(uint64_t seed, uint64_t gid, uint64_t w) {
  uint64_t x = (gid * 0x9E3779B97F4A7C15ULL) ^ (w * 0xD6E8FEB86659FD93ULL) ^ seed;
  x ^= x >> 32;
  x *= 0xD6E8FEB86659FD93ULL;
  x ^= x >> 32;
  return static_cast<uint32_t>(x);
}
__device__ __forceinline__ uint32_t synth_label(uint64_t seed, uint64_t gid, uint32_t n_labels) {
  return static_cast<uint32_t>(mix64_step(seed, gid) % n_labels);
}
// byte b (b >= 8) of record gid
__device__ __forceinline__ uint8_t synth_byte(uint64_t seed, uint64_t gid, uint64_t b) {
  return static_cast<uint8_t>(synth_word(seed, gid, (b - 8) >> 2) >> (8 * ((b - 8) & 3)));
}

__global__ void synth_index_kernel(uint64_t* off, uint32_t* len, uint32_t* label, int64_t n,
                                   int64_t rec_bytes, int64_t first_gid, int64_t stride,
                                   uint64_t seed, uint32_t n_labels) {
  int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= n) return;
  uint64_t gid = static_cast<uint64_t>(first_gid + j * stride);
  off[j] = static_cast<uint64_t>(j) * rec_bytes;
  len[j] = static_cast<uint32_t>(rec_bytes);
  label[j] = synth_label(seed, gid, n_labels);
}

// one CTA per record (grid-stride); records are 16-byte aligned when
// rec_bytes % 16 == 0 (the 224x224x3 case), else the byte path runs
__global__ void __launch_bounds__(512) synth_blob_kernel(uint8_t* blob, int64_t n,
                                                         int64_t rec_bytes, int64_t first_gid,
                                                         int64_t stride, uint64_t seed) {
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    uint64_t gid = static_cast<uint64_t>(first_gid + j * stride);
    uint8_t* rec = blob + j * rec_bytes;
    if ((rec_bytes & 15) == 0) {
      uint4* r4 = reinterpret_cast<uint4*>(rec);
      int64_t nv = rec_bytes / 16;
      for (int64_t k = threadIdx.x; k < nv; k += blockDim.x) {
        uint4 x;
        if (k == 0) {
          x.x = static_cast<uint32_t>(gid);
          x.y = static_cast<uint32_t>(gid >> 32);
          x.z = synth_word(seed, gid, 0);
          x.w = synth_word(seed, gid, 1);
        } else {
          uint64_t w0 = 4 * k - 2;
          x.x = synth_word(seed, gid, w0);
          x.y = synth_word(seed, gid, w0 + 1);
          x.z = synth_word(seed, gid, w0 + 2);
          x.w = synth_word(seed, gid, w0 + 3);
        }
        __stcs(r4 + k, x);
      }
    } else {
      for (int64_t b = threadIdx.x; b < rec_bytes; b += blockDim.x)
        rec[b] = b < 8 ? static_cast<uint8_t>(gid >> (8 * b)) : synth_byte(seed, gid, b);
    }
  }
}

__global__ void __launch_bounds__(512) synth_verify_kernel(const uint8_t* blob,
                                                           const uint64_t* off,
                                                           const uint32_t* len,
                                                           const uint32_t* label, int64_t n,
                                                           uint64_t seed, uint32_t n_labels,
                                                           unsigned long long* gids,
                                                           unsigned long long* bad) {
  __shared__ int s_bad;
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    const uint8_t* rec = blob + off[j];
    uint32_t L = len[j];
    if (threadIdx.x == 0) s_bad = L < 8;
    __syncthreads();
    if (L >= 8) {
      uint64_t gid = 0;
      for (int b = 7; b >= 0; --b) gid = (gid << 8) | rec[b];
      if (threadIdx.x == 0) {
        if (gids) gids[j] = gid;
        if (label[j] != synth_label(seed, gid, n_labels)) s_bad = 1;
      }
      int mism = 0;
      for (uint64_t b = 8 + threadIdx.x; b < L; b += blockDim.x)
        mism |= rec[b] != synth_byte(seed, gid, b);
      if (mism) s_bad = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_bad) atomicAdd(bad, 1ULL);
    __syncthreads();
  }
}

static int blocks_for(int64_t n, int t = 256) {
  int64_t b = (n + t - 1) / t;
  return static_cast<int>(b < 1 ? 1 : (b > (1LL << 30) ? (1LL << 30) : b));
}

// The shuffle's exchange kernels: 2 CTAs x 512 threads per SM keep the links
// saturated (each CTA has 32 KB of 16-byte loads in flight) and leave every SM
// room for the next epoch's plan kernels on a side stream (shuffle_all's
// next_seed).
static int exchange_grid(int64_t n) {
  int dev = 0;
  cudaGetDevice(&dev);
  int64_t cap = static_cast<int64_t>(sm_count(dev)) * 2;
  return static_cast<int>(n < 1 ? 1 : (n < cap ? n : cap));
}

// Record-copy grids (gather, synthetic corpus): up to 8 CTAs of 512 threads
// per SM, i.e. two waves of resident CTAs -- the second wave evens out the
// per-CTA unit counts (tools/gather_variants.cu, 8,192 random 150 KB records:
// 5.89 TB/s with 4 CTAs per SM, 6.39 TB/s with 8; cudaMemcpy of the same
// bytes 6.49 TB/s).
static int record_grid(int64_t n) {
  int dev = 0;
  cudaGetDevice(&dev);
  int64_t cap = static_cast<int64_t>(sm_count(dev)) * 8;
  return static_cast<int>(n < 1 ? 1 : (n < cap ? n : cap));
}

}  // namespace md

using namespace md;

extern "C" {

uint64_t md_mix64(const uint64_t* parts, int32_t n) {
  uint64_t acc = 0;
  for (int i = 0; i < n; ++i) acc = mix64_step(acc, parts[i]);
  return acc;
}

int md_random_batch(uint64_t key, int64_t n_records, int64_t batch, int64_t* picks, void* stream) {
  if (n_records <= 0) {
    set_error("cannot sample from an empty shard");
    return MD_ERR_EMPTY_SHARD;
  }
  if (batch < 1) {
    set_error("batch_size must be >= 1, got %lld", (long long)batch);
    return MD_ERR_INVALID_CONFIG;
  }
  if (n_records > 0xFFFFFFFFLL) {
    set_error("shards above 2^32 records are not supported");
    return MD_ERR_INVALID_CONFIG;
  }
  cudaStream_t s = as_stream(stream);
  if (batch <= 1024) {  // one CTA: rejection detected with a block vote, no scratch
    picks_block_kernel<<<1, 1024, 0, s>>>(key, static_cast<uint32_t>(n_records), batch, picks);
    MD_LAUNCH_CHECK();
    return MD_OK;
  }
  int* bad = nullptr;
  MD_CUDA_TRY(cudaMallocAsync(&bad, sizeof(int), s));
  MD_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), s));
  picks_kernel<<<blocks_for(batch), 256, 0, s>>>(key, static_cast<uint32_t>(n_records), batch,
                                                 picks, bad);
  MD_LAUNCH_CHECK();
  if (n_records > 1) {
    picks_fix_kernel<<<1, 1024, 0, s>>>(key, static_cast<uint32_t>(n_records), batch, picks, bad);
    MD_LAUNCH_CHECK();
  }
  MD_CUDA_TRY(cudaFreeAsync(bad, s));
  return MD_OK;
}

int md_random_batch_step(uint64_t seed, uint64_t role, uint64_t worker, int64_t* step,
                         int64_t n_records, int64_t batch, int64_t* picks, void* stream) {
  if (n_records <= 0) {
    set_error("cannot sample from an empty shard");
    return MD_ERR_EMPTY_SHARD;
  }
  if (batch < 1 || batch > 1024 || n_records > 0xFFFFFFFFLL) {
    set_error("md_random_batch_step needs 1 <= batch <= 1024 and < 2^32 records");
    return MD_ERR_INVALID_CONFIG;
  }
  static std::atomic<uint64_t> carve{0};
  prefer_max_smem(picks_step_kernel, carve);
  picks_step_kernel<<<1, 1024, 0, as_stream(stream)>>>(seed, role, worker, step,
                                                      static_cast<uint32_t>(n_records), batch, picks);
  MD_LAUNCH_CHECK();
  return MD_OK;
}

int md_gather(const uint8_t* blob, const uint64_t* off, const uint32_t* len, const uint32_t* label,
              const int64_t* picks, int64_t batch, uint8_t* out, int64_t out_stride,
              const uint64_t* out_off, uint32_t* out_label, int32_t* err_flag, void* stream) {
  if (batch <= 0) return MD_OK;
  if (out_stride == 0 && !out_off) {
    set_error("packed gather needs out_off");
    return MD_ERR_INVALID_CONFIG;
  }
  const int chunks =
      out_stride > 0 ? static_cast<int>((out_stride + kGatherChunk - 1) / kGatherChunk) : 1;
  int dev = 0;
  MD_CUDA_TRY(cudaGetDevice(&dev));
  const int64_t units = batch * chunks;
  if (units <= static_cast<int64_t>(sm_count(dev)) * 2) {  // a training-step batch
    static std::atomic<uint64_t> carve{0};
    prefer_max_smem(gather_kernel<true>, carve);
    gather_kernel<true><<<record_grid(units), 512, 0, as_stream(stream)>>>(
        blob, off, len, label, picks, batch, out, out_stride, out_off, out_label, err_flag, chunks);
  } else {
    gather_kernel<false><<<record_grid(units), 512, 0, as_stream(stream)>>>(
        blob, off, len, label, picks, batch, out, out_stride, out_off, out_label, err_flag, chunks);
  }
  MD_LAUNCH_CHECK();
  return MD_OK;
}

// MD_DIMD_TIMING=1: synchronize and print the wall time of each plan phase
struct PlanTimer {
  cudaStream_t s;
  bool on;
  std::chrono::steady_clock::time_point t;
  static bool enabled() {
    static const bool on = getenv("MD_DIMD_TIMING") != nullptr;  // read once
    return on;
  }
  explicit PlanTimer(cudaStream_t st) : s(st), on(enabled()) {
    t = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[md_shuffle_plan] %-12s %8.3f ms\n", what,
            std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

int md_shuffle_plan(uint64_t seed, uint64_t group_id, int32_t S, int32_t member,
                    uint64_t global_rank, int64_t m_segments, const int64_t* n_rec,
                    int32_t* final_member, int64_t* final_rec, int64_t cap, int64_t* n_final,
                    int64_t* next_counts, void* stream) {
  if (S < 1 || S > MD_MAX_GROUP || member < 0 || member >= S) {
    set_error("bad group shape S=%d member=%d (max group %d)", S, member, MD_MAX_GROUP);
    return MD_ERR_INVALID_CONFIG;
  }
  if (m_segments < 1) {
    set_error("m_segments must be >= 1, got %lld", (long long)m_segments);
    return MD_ERR_INVALID_CONFIG;
  }
  SrcTable tab;
  memset(&tab, 0, sizeof(tab));
  int64_t total = 0;
  for (int q = 0; q < S; ++q) {
    if (n_rec[q] < 0 || n_rec[q] > 0x7FFFFFFFLL) {
      set_error("member %d holds %lld records (limit 2^31-1)", q, (long long)n_rec[q]);
      return MD_ERR_INVALID_CONFIG;
    }
    tab.n_rec[q] = n_rec[q];
    tab.base[q] = total;
    total += n_rec[q];
  }
  for (int q = S; q <= MD_MAX_GROUP; ++q) tab.base[q] = total;
  cudaStream_t s = as_stream(stream);
  const int64_t m = m_segments;
  PlanTimer pt(s);
  {  // keep the stream-ordered pool's memory between calls (no re-growth per plan)
    static std::atomic<uint64_t> pool_set{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !(pool_set.fetch_or(1ull << dev) & (1ull << dev))) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
    }
  }

  int32_t *dest = nullptr, *flag = nullptr, *excl = nullptr, *got_m = nullptr;
  int64_t *got_r = nullptr, *base_tq = nullptr, *d_nf = nullptr;
  unsigned long long* d_cnt = nullptr;
  uint8_t* seg_bad = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  const int64_t tot1 = total + 1;
  MD_CUDA_TRY(cudaMallocAsync(&dest, sizeof(int32_t) * (total + 1), s));
  MD_CUDA_TRY(cudaMallocAsync(&flag, sizeof(int32_t) * tot1, s));
  MD_CUDA_TRY(cudaMallocAsync(&excl, sizeof(int32_t) * tot1, s));
  MD_CUDA_TRY(cudaMallocAsync(&seg_bad, S * m, s));
  MD_CUDA_TRY(cudaMallocAsync(&base_tq, sizeof(int64_t) * S * m, s));
  MD_CUDA_TRY(cudaMallocAsync(&d_nf, sizeof(int64_t), s));
  MD_CUDA_TRY(cudaMallocAsync(&d_cnt, sizeof(unsigned long long) * MD_MAX_GROUP, s));
  MD_CUDA_TRY(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * MD_MAX_GROUP, s));
  MD_CUDA_TRY(cudaMemsetAsync(seg_bad, 0, S * m, s));
  MD_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int32_t) * tot1, s));
  if (total > 0) {
    dest_kernel<<<blocks_for(total), 256, 0, s>>>(tab, S, m, seed, group_id, total, dest, seg_bad);
    MD_LAUNCH_CHECK();
    if (S > 1 && (S & (S - 1)) != 0) {  // only non-powers of two can reject
      dest_fix_kernel<<<blocks_for(S * m), 256, 0, s>>>(tab, S, m, seed, group_id, dest, seg_bad);
      MD_LAUNCH_CHECK();
    }
    mine_flag_kernel<<<blocks_for(total), 256, 0, s>>>(dest, total, member, flag);
    MD_LAUNCH_CHECK();
    if (next_counts) {
      dest_count_kernel<<<std::min(blocks_for(total), 1024), 256, 0, s>>>(dest, total, S, d_cnt);
      MD_LAUNCH_CHECK();
    }
  }
  pt.mark("dest draws");
  MD_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, flag, excl, tot1, s));
  MD_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, s));
  MD_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flag, excl, tot1, s));
  MD_CUDA_TRY(cudaFreeAsync(tmp, s));
  recv_base_kernel<<<1, 1, 0, s>>>(tab, S, m, excl, base_tq, d_nf);
  MD_LAUNCH_CHECK();
  int64_t nf = 0;
  unsigned long long cnt_h[MD_MAX_GROUP] = {0};
  MD_CUDA_TRY(cudaMemcpyAsync(&nf, d_nf, sizeof(nf), cudaMemcpyDeviceToHost, s));
  if (next_counts)
    MD_CUDA_TRY(cudaMemcpyAsync(cnt_h, d_cnt, sizeof(unsigned long long) * S,
                                cudaMemcpyDeviceToHost, s));
  MD_CUDA_TRY(cudaFreeAsync(d_cnt, s));
  MD_CUDA_TRY(cudaStreamSynchronize(s));
  if (next_counts)
    for (int q = 0; q < S; ++q) next_counts[q] = static_cast<int64_t>(cnt_h[q]);
  if (nf > cap) {
    set_error("shuffle output of %lld records exceeds capacity %lld", (long long)nf,
              (long long)cap);
    return MD_ERR_INVALID_CONFIG;
  }
  MD_CUDA_TRY(cudaMallocAsync(&got_m, sizeof(int32_t) * (nf + 1), s));
  MD_CUDA_TRY(cudaMallocAsync(&got_r, sizeof(int64_t) * (nf + 1), s));
  if (total > 0) {
    got_scatter_kernel<<<blocks_for(total), 256, 0, s>>>(tab, S, m, total, flag, excl, base_tq,
                                                         got_m, got_r);
    MD_LAUNCH_CHECK();
  }
  MD_CUDA_TRY(cudaFreeAsync(dest, s));
  MD_CUDA_TRY(cudaFreeAsync(flag, s));
  MD_CUDA_TRY(cudaFreeAsync(excl, s));
  MD_CUDA_TRY(cudaFreeAsync(seg_bad, s));
  MD_CUDA_TRY(cudaFreeAsync(base_tq, s));
  MD_CUDA_TRY(cudaFreeAsync(d_nf, s));
  pt.mark("recv order");

  // ---- permutation(nf), key _mix64(seed, "perm", global_rank)
  uint64_t parts[3] = {seed, kRolePerm, global_rank};
  const uint64_t pkey = md_mix64(parts, 3);
  if (nf > 0xFFFFFFFFLL) {
    set_error("permutation of more than 2^32 records unsupported");
    return MD_ERR_INVALID_CONFIG;
  }
  if (nf <= 1) {
    if (nf == 1) {
      MD_CUDA_TRY(cudaMemcpyAsync(final_member, got_m, sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
      MD_CUDA_TRY(cudaMemcpyAsync(final_rec, got_r, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    }
  } else {
    const int64_t steps = nf - 1;  // s = nf-1 .. 1
    uint32_t *J = nullptr, *ws = nullptr, *tgt = nullptr, *stp = nullptr, *tgt_s = nullptr,
             *stp_s = nullptr;
    int32_t *nxt = nullptr, *parent = nullptr, *pa = nullptr, *pb = nullptr;
    int64_t* st = nullptr;
    int* changed = nullptr;
    MD_CUDA_TRY(cudaMallocAsync(&J, sizeof(uint32_t) * nf, s));
    MD_CUDA_TRY(cudaMallocAsync(&st, sizeof(int64_t) * 2, s));
    int64_t st_h[2] = {steps, 0};
    MD_CUDA_TRY(cudaMemcpyAsync(st, st_h, sizeof(st_h), cudaMemcpyHostToDevice, s));
    int64_t chunk = 2 * nf + 4096, word_base = 0;
    MD_CUDA_TRY(cudaMallocAsync(&ws, sizeof(uint32_t) * (chunk + 64), s));
    while (true) {
      words_kernel<<<blocks_for(chunk + 64), 256, 0, s>>>(pkey, word_base, chunk + 64, ws);
      MD_LAUNCH_CHECK();
      pt.mark("fy gen");
      fy_scan_kernel<<<1, 32, 0, s>>>(ws, chunk + 64, word_base, J, st);
      MD_LAUNCH_CHECK();
      pt.mark("fy scan");
      MD_CUDA_TRY(cudaMemcpyAsync(st_h, st, sizeof(st_h), cudaMemcpyDeviceToHost, s));
      MD_CUDA_TRY(cudaStreamSynchronize(s));
      if (st_h[0] == 0) break;
      word_base = st_h[1];  // resume at the first unconsumed word
    }
    MD_CUDA_TRY(cudaFreeAsync(ws, s));
    pt.mark("fy words");
    MD_CUDA_TRY(cudaMallocAsync(&tgt_s, sizeof(uint32_t) * steps, s));
    MD_CUDA_TRY(cudaMallocAsync(&stp, sizeof(uint32_t) * steps, s));
    MD_CUDA_TRY(cudaMallocAsync(&stp_s, sizeof(uint32_t) * steps, s));
    iota_kernel<<<blocks_for(steps), 256, 0, s>>>(stp, steps, 1u);
    MD_LAUNCH_CHECK();
    tgt = J + 1;  // J[1..nf-1]
    int end_bit = 1;
    while (end_bit < 32 && (1LL << end_bit) < nf) ++end_bit;
    tmp_bytes = 0;
    MD_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, tgt, tgt_s, stp, stp_s,
                                                 static_cast<int>(steps), 0, end_bit, s));
    MD_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, s));
    MD_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, tgt, tgt_s, stp, stp_s,
                                                 static_cast<int>(steps), 0, end_bit, s));
    MD_CUDA_TRY(cudaFreeAsync(tmp, s));
    pt.mark("fy sort");
    MD_CUDA_TRY(cudaMallocAsync(&nxt, sizeof(int32_t) * nf, s));
    MD_CUDA_TRY(cudaMallocAsync(&parent, sizeof(int32_t) * nf, s));
    MD_CUDA_TRY(cudaMallocAsync(&pa, sizeof(int32_t) * nf, s));
    MD_CUDA_TRY(cudaMallocAsync(&pb, sizeof(int32_t) * nf, s));
    MD_CUDA_TRY(cudaMallocAsync(&changed, sizeof(int), s));
    fill_i32_kernel<<<blocks_for(nf), 256, 0, s>>>(nxt, nf, -1);
    MD_LAUNCH_CHECK();
    fill_i32_kernel<<<blocks_for(nf), 256, 0, s>>>(parent, nf, -1);
    MD_LAUNCH_CHECK();
    fy_links_kernel<<<blocks_for(steps), 256, 0, s>>>(tgt_s, stp_s, steps, nxt, parent);
    MD_LAUNCH_CHECK();
    ptr_init_kernel<<<blocks_for(nf), 256, 0, s>>>(parent, nf, pa);
    MD_LAUNCH_CHECK();
    // pointer jumping: chains are at most nf long -> ceil(log2 nf) + 1 rounds
    int rounds = 1;
    while ((1LL << rounds) < nf) ++rounds;
    for (int r = 0; r <= rounds; ++r) {
      ptr_jump_kernel<<<blocks_for(nf), 256, 0, s>>>(pa, nf, pb, changed);
      MD_LAUNCH_CHECK();
      std::swap(pa, pb);
    }
    fy_final_kernel<<<blocks_for(nf), 256, 0, s>>>(nxt, pa, J, tgt_s, stp_s, nf, got_m, got_r,
                                                  final_member, final_rec);
    MD_LAUNCH_CHECK();
    for (void* p : {(void*)J, (void*)tgt_s, (void*)stp, (void*)stp_s, (void*)nxt, (void*)parent,
                    (void*)pa, (void*)pb, (void*)changed, (void*)st})
      MD_CUDA_TRY(cudaFreeAsync(p, s));
  }
  MD_CUDA_TRY(cudaFreeAsync(got_m, s));
  MD_CUDA_TRY(cudaFreeAsync(got_r, s));
  pt.mark("fy resolve");
  *n_final = nf;
  return MD_OK;
}

int md_shuffle_index(int32_t S, const uint32_t* const* peer_len, const uint32_t* const* peer_label,
                     const int32_t* final_member, const int64_t* final_rec, int64_t n_final,
                     uint64_t* out_off, uint32_t* out_len, uint32_t* out_label,
                     uint64_t* total_bytes, void* stream) {
  if (S < 1 || S > MD_MAX_GROUP) {
    set_error("bad group size %d", S);
    return MD_ERR_INVALID_CONFIG;
  }
  *total_bytes = 0;
  if (n_final == 0) return MD_OK;
  cudaStream_t s = as_stream(stream);
  PeerIdx p;
  memset(&p, 0, sizeof(p));
  for (int q = 0; q < S; ++q) {
    p.len[q] = peer_len[q];
    p.label[q] = peer_label[q];
  }
  unsigned long long* len64 = nullptr;
  MD_CUDA_TRY(cudaMallocAsync(&len64, sizeof(unsigned long long) * (n_final + 1), s));
  MD_CUDA_TRY(cudaMemsetAsync(len64 + n_final, 0, sizeof(unsigned long long), s));
  index_kernel<<<blocks_for(n_final), 256, 0, s>>>(p, final_member, final_rec, n_final, out_len,
                                                   out_label, len64);
  MD_LAUNCH_CHECK();
  unsigned long long* offs = nullptr;
  MD_CUDA_TRY(cudaMallocAsync(&offs, sizeof(unsigned long long) * (n_final + 1), s));
  void* tmp = nullptr;
  size_t tb = 0;
  MD_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, len64, offs, n_final + 1, s));
  MD_CUDA_TRY(cudaMallocAsync(&tmp, tb, s));
  MD_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, len64, offs, n_final + 1, s));
  MD_CUDA_TRY(cudaMemcpyAsync(out_off, offs, sizeof(uint64_t) * n_final, cudaMemcpyDeviceToDevice, s));
  unsigned long long tot = 0;
  MD_CUDA_TRY(cudaMemcpyAsync(&tot, offs + n_final, sizeof(tot), cudaMemcpyDeviceToHost, s));
  MD_CUDA_TRY(cudaFreeAsync(tmp, s));
  MD_CUDA_TRY(cudaFreeAsync(offs, s));
  MD_CUDA_TRY(cudaFreeAsync(len64, s));
  MD_CUDA_TRY(cudaStreamSynchronize(s));
  *total_bytes = tot;
  return MD_OK;
}

int md_shuffle_pull(int32_t S, const uint8_t* const* peer_blob, const uint64_t* const* peer_off,
                    const int32_t* final_member, const int64_t* final_rec, int64_t n_final,
                    const uint64_t* out_off, const uint32_t* out_len, uint8_t* out_blob,
                    void* stream) {
  if (S < 1 || S > MD_MAX_GROUP) {
    set_error("bad group size %d", S);
    return MD_ERR_INVALID_CONFIG;
  }
  if (n_final == 0) return MD_OK;
  PeerBlob p;
  memset(&p, 0, sizeof(p));
  for (int q = 0; q < S; ++q) {
    p.blob[q] = peer_blob[q];
    p.off[q] = peer_off[q];
  }
  pull_kernel<<<exchange_grid(n_final), 512, 0, as_stream(stream)>>>(
      p, final_member, final_rec, n_final, out_off, out_len, out_blob);
  MD_LAUNCH_CHECK();
  return MD_OK;
}

int md_shuffle_sendlist(int32_t S, const int32_t* final_member, const int64_t* final_rec,
                        int64_t n_final, const uint64_t* out_off, const uint32_t* out_len,
                        void* list, int64_t* begin, void* stream) {
  if (S < 1 || S > MD_MAX_GROUP) {
    set_error("bad group size %d", S);
    return MD_ERR_INVALID_CONFIG;
  }
  if (n_final > 0x7FFFFFFFLL) {
    set_error("send list of more than 2^31 records unsupported");
    return MD_ERR_INVALID_CONFIG;
  }
  cudaStream_t s = as_stream(stream);
  unsigned long long* cnt = nullptr;
  MD_CUDA_TRY(cudaMallocAsync(&cnt, sizeof(unsigned long long) * MD_MAX_GROUP, s));
  MD_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * MD_MAX_GROUP, s));
  if (n_final > 0) {
    member_count_kernel<<<std::min(blocks_for(n_final), 1024), 256, 0, s>>>(final_member, n_final,
                                                                           S, cnt);
    MD_LAUNCH_CHECK();
  }
  member_begin_kernel<<<1, 1, 0, s>>>(cnt, S, begin);
  MD_LAUNCH_CHECK();
  MD_CUDA_TRY(cudaFreeAsync(cnt, s));
  if (n_final == 0) return MD_OK;
  // stable sort of slot ids by source member (slot order kept per member)
  const int n = static_cast<int>(n_final);
  int32_t *ids = nullptr, *ids_s = nullptr, *keys_s = nullptr;
  MD_CUDA_TRY(cudaMallocAsync(&ids, sizeof(int32_t) * n, s));
  MD_CUDA_TRY(cudaMallocAsync(&ids_s, sizeof(int32_t) * n, s));
  MD_CUDA_TRY(cudaMallocAsync(&keys_s, sizeof(int32_t) * n, s));
  iota_kernel<<<blocks_for(n), 256, 0, s>>>(reinterpret_cast<uint32_t*>(ids), n, 0u);
  MD_LAUNCH_CHECK();
  int end_bit = 1;
  while ((1 << end_bit) < S) ++end_bit;
  size_t tb = 0;
  void* tmp = nullptr;
  MD_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, final_member, keys_s, ids, ids_s, n, 0,
                                               end_bit, s));
  MD_CUDA_TRY(cudaMallocAsync(&tmp, tb, s));
  MD_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, final_member, keys_s, ids, ids_s, n, 0,
                                               end_bit, s));
  sendlist_kernel<<<blocks_for(n), 256, 0, s>>>(ids_s, final_member, final_rec, out_off, out_len,
                                                n, static_cast<SendEntry*>(list));
  MD_LAUNCH_CHECK();
  for (void* p : {tmp, (void*)ids, (void*)ids_s, (void*)keys_s}) MD_CUDA_TRY(cudaFreeAsync(p, s));
  return MD_OK;
}

int md_shuffle_push(int32_t S, int32_t member, const uint8_t* blob, const uint64_t* off,
                    const void* const* peer_list, const int64_t* const* peer_begin,
                    uint8_t* const* peer_out, void* stream) {
  if (S < 1 || S > MD_MAX_GROUP || member < 0 || member >= S) {
    set_error("bad group shape S=%d member=%d", S, member);
    return MD_ERR_INVALID_CONFIG;
  }
  PushArgs p;
  memset(&p, 0, sizeof(p));
  for (int d = 0; d < S; ++d) {
    p.list[d] = static_cast<const SendEntry*>(peer_list[d]);
    p.begin[d] = peer_begin[d];
    p.out[d] = peer_out[d];
  }
  // (work items are records, many per CTA: the full exchange grid; a
  // one-member group only copies within its own HBM, where the record-copy
  // grid's second wave of CTAs evens out the tail)
  if (S == 1)
    push_kernel<true><<<record_grid(INT64_MAX), 512, 0, as_stream(stream)>>>(p, S, member, blob, off);
  else
    push_kernel<false><<<exchange_grid(INT64_MAX), 512, 0, as_stream(stream)>>>(p, S, member, blob,
                                                                               off);
  MD_LAUNCH_CHECK();
  return MD_OK;
}

int md_copy_segments(int32_t n_seg, uint8_t* const* dst, const uint8_t* const* src,
                     const uint64_t* len, void* stream) {
  if (n_seg < 0 || n_seg > MD_MAX_GROUP) {
    set_error("%d segments exceed the limit %d", n_seg, MD_MAX_GROUP);
    return MD_ERR_INVALID_CONFIG;
  }
  SegCopy p;
  memset(&p, 0, sizeof(p));
  uint64_t blocks = 0;
  for (int i = 0; i < n_seg; ++i) {
    p.dst[i] = dst[i];
    p.src[i] = src[i];
    p.len[i] = len[i];
    p.blocks_before[i] = blocks;
    blocks += (len[i] + kSliceBytes - 1) / kSliceBytes;
  }
  p.blocks_before[n_seg] = blocks;
  if (blocks == 0) return MD_OK;
  if (blocks > (1u << 31) - 1) {
    set_error("copy too large");
    return MD_ERR_INVALID_CONFIG;
  }
  segcopy_kernel<<<static_cast<unsigned>(blocks), 512, 0, as_stream(stream)>>>(p, n_seg);
  MD_LAUNCH_CHECK();
  return MD_OK;
}

int md_synth_records(uint8_t* blob, uint64_t* off, uint32_t* len, uint32_t* label, int64_t n_local,
                     int64_t rec_bytes, int64_t first_gid, int64_t gid_stride, uint64_t seed,
                     uint32_t n_labels, void* stream) {
  if (rec_bytes < 8 || rec_bytes >= (1LL << 31) || n_labels == 0) {
    set_error("synthetic records need 8 <= rec_bytes < 2^31 and n_labels >= 1");
    return MD_ERR_INVALID_CONFIG;
  }
  if (n_local <= 0) return MD_OK;
  cudaStream_t s = as_stream(stream);
  synth_index_kernel<<<blocks_for(n_local), 256, 0, s>>>(off, len, label, n_local, rec_bytes,
                                                         first_gid, gid_stride, seed, n_labels);
  MD_LAUNCH_CHECK();
  synth_blob_kernel<<<record_grid(n_local), 512, 0, s>>>(blob, n_local, rec_bytes, first_gid,
                                                        gid_stride, seed);
  MD_LAUNCH_CHECK();
  return MD_OK;
}

int md_synth_verify(const uint8_t* blob, const uint64_t* off, const uint32_t* len,
                    const uint32_t* label, int64_t n, uint64_t seed, uint32_t n_labels,
                    uint64_t* gids, int64_t* n_bad, void* stream) {
  *n_bad = 0;
  if (n <= 0) return MD_OK;
  cudaStream_t s = as_stream(stream);
  unsigned long long* bad = nullptr;
  MD_CUDA_TRY(cudaMallocAsync(&bad, sizeof(*bad), s));
  MD_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(*bad), s));
  synth_verify_kernel<<<record_grid(n), 512, 0, s>>>(blob, off, len, label, n, seed, n_labels,
                                                    reinterpret_cast<unsigned long long*>(gids),
                                                    bad);
  MD_LAUNCH_CHECK();
  unsigned long long h = 0;
  MD_CUDA_TRY(cudaMemcpyAsync(&h, bad, sizeof(h), cudaMemcpyDeviceToHost, s));
  MD_CUDA_TRY(cudaFreeAsync(bad, s));
  MD_CUDA_TRY(cudaStreamSynchronize(s));
  *n_bad = static_cast<int64_t>(h);
  return MD_OK;
}

}  // extern "C"
