// Shared device/host helpers for libmdb200 (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "../../include/mdb200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libmdb200 is written for sm_100a (B200) only"
#endif

namespace md {

// ---- error plumbing (host) --------------------------------------------------
void set_error(const char* fmt, ...);
extern std::atomic<uint64_t> g_launches;

#define MD_CUDA_TRY(expr)                                                                  \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess) {                                                               \
      md::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__,       \
                    __LINE__);                                                             \
      return MD_ERR_CUDA;                                                                  \
    }                                                                                      \
  } while (0)

#define MD_LAUNCH_CHECK()                                                                  \
  do {                                                                                     \
    md::g_launches.fetch_add(1, std::memory_order_relaxed);                                \
    cudaError_t _e = cudaGetLastError();                                                   \
    if (_e != cudaSuccess) {                                                               \
      md::set_error("kernel launch failed: %s (%s:%d)", cudaGetErrorString(_e), __FILE__,   \
                    __LINE__);                                                             \
      return MD_ERR_CUDA;                                                                  \
    }                                                                                      \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// The kernels that run back to back with the allreduce in a training step ask
// for the max-shared carveout too, so the SM does not re-partition L1/SMEM
// (a drain) between them and the 192 KB-SMEM allreduce. Once per device;
// MD_DEFAULT_CARVEOUT=1 leaves the driver default (A/B switch).
template <class K>
inline void prefer_max_smem(K kernel, std::atomic<uint64_t>& done) {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) return;
  const uint64_t bit = 1ull << (d & 63);
  if (done.load(std::memory_order_relaxed) & bit) return;
  if (!getenv("MD_DEFAULT_CARVEOUT"))
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
  done.fetch_or(bit);
}

int sm_count(int device);

// ---- exact float32 arithmetic (no contraction: every op rounds once) --------
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                     __fadd_rn(a.w, b.w));
}

// SGD update of one element, the contract of md_sgd_update (mdb200.h).
template <bool kWd, bool kMom>
__device__ __forceinline__ void sgd1(float& w, float g, float* v, float c, float mu, float wd_b) {
  float d = g;
  if (kWd) d = __fadd_rn(g, __fmul_rn(wd_b, w));
  if (kMom) {
    float nv = __fadd_rn(__fmul_rn(mu, *v), d);
    *v = nv;
    d = nv;
  }
  w = __fsub_rn(w, __fmul_rn(c, d));
}

// ---- memory-model helpers for the cross-GPU epoch protocol ------------------
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_sys64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_sys() {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// ---- TMA (cp.async.bulk, 1-D) + mbarrier ---------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
      : "=r"(done)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return done != 0;
}
// global (local or NVLink-peer address) -> shared, completion on `bar`
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
// generic-proxy writes/acquires -> async-proxy (TMA) reads of global memory
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// epoch comparison robust to 32-bit wrap: a >= b
__device__ __forceinline__ bool epoch_ge(uint32_t a, uint32_t b) {
  return static_cast<int32_t>(a - b) >= 0;
}

// ---- Philox4x64-10 (numpy's bit generator) ----------------------------------
// numpy/random/src/philox: counter incremented before each block, key =
// (seed mod 2^64, seed >> 64); round multipliers on v0 and v2.
struct U64x4 {
  uint64_t v[4];
};

__host__ __device__ __forceinline__ void mulhilo64(uint64_t a, uint64_t b, uint64_t* hi,
                                                   uint64_t* lo) {
#if defined(__CUDA_ARCH__)
  *lo = a * b;
  *hi = __umul64hi(a, b);
#else
  unsigned __int128 p = static_cast<unsigned __int128>(a) * b;
  *lo = static_cast<uint64_t>(p);
  *hi = static_cast<uint64_t>(p >> 64);
#endif
}

// Block for 256-bit counter (c0, c1, 0, 0) -- counters here never exceed 2^64.
__host__ __device__ __forceinline__ U64x4 philox4x64_10(uint64_t c0, uint64_t c1, uint64_t k0,
                                                        uint64_t k1) {
  uint64_t v0 = c0, v1 = c1, v2 = 0, v3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ULL, v0, &hi0, &lo0);
    mulhilo64(0xCA5A826395121157ULL, v2, &hi1, &lo1);
    uint64_t n0 = hi1 ^ v1 ^ k0;
    uint64_t n2 = hi0 ^ v3 ^ k1;
    v0 = n0;
    v1 = lo1;
    v2 = n2;
    v3 = lo0;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  U64x4 o;
  o.v[0] = v0;
  o.v[1] = v1;
  o.v[2] = v2;
  o.v[3] = v3;
  return o;
}

// 32-bit word `w` of the stream of a fresh Generator(Philox(key)):
// u64 index w/2 (low half first), block (w/2)/4, counter = block + 1.
__host__ __device__ __forceinline__ uint32_t philox_word32(uint64_t key, uint64_t w) {
  uint64_t q = w >> 1;
  uint64_t blk = q >> 2;
  U64x4 b = philox4x64_10(blk + 1, 0, key, 0);
  uint64_t x = b.v[q & 3];
  return (w & 1) ? static_cast<uint32_t>(x >> 32) : static_cast<uint32_t>(x);
}

// splitmix-style key mixer, dimd.py:226-234
__host__ __device__ __forceinline__ uint64_t mix64_step(uint64_t acc, uint64_t p) {
  acc = acc + p + 0x9E3779B97F4A7C15ULL;
  acc = (acc ^ (acc >> 30)) * 0xBF58476D1CE4E5B9ULL;
  acc = (acc ^ (acc >> 27)) * 0x94D049BB133111EBULL;
  acc ^= acc >> 31;
  return acc;
}

}  // namespace md
