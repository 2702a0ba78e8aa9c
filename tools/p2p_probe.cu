// p2p_probe: peer-read bandwidth on B200 NVLink, three ways, GPU b reading
// GPU a's HBM (and both directions at once):
//   ldg   - float4 loads from the peer pointer (U per thread) + local stores
//   bulk  - cp.async.bulk (TMA, 1-D) peer -> shared (mbarrier pipeline) ->
//           cp.async.bulk shared -> local global
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/p2p_probe tools/p2p_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));     \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

template <int U>
__global__ void __launch_bounds__(512) ldg_copy(const float4* __restrict__ src,
                                                float4* __restrict__ dst, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t b = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; b < n; b += stride) {
    float4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (b + (size_t)u * blockDim.x < n) x[u] = src[b + (size_t)u * blockDim.x];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (b + (size_t)u * blockDim.x < n) dst[b + (size_t)u * blockDim.x] = x[u];
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int NS>
__global__ void __launch_bounds__(128) bulk_copy(const char* __restrict__ src,
                                                 char* __restrict__ dst, size_t bytes,
                                                 int chunk) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t full[NS];
  // contiguous slice per CTA
  size_t per = (bytes / gridDim.x + 15) & ~size_t(15);
  size_t lo = per * blockIdx.x, hi = lo + per < bytes ? lo + per : bytes;
  if (lo >= hi) return;
  int nchunks = (int)((hi - lo + chunk - 1) / chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  auto issue = [&](int c) {
    int s = c % NS;
    size_t off = lo + (size_t)c * chunk;
    uint32_t nb = (uint32_t)((hi - off) < (size_t)chunk ? (hi - off) : chunk);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                 "r"(nb)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem + (size_t)s * chunk)),
        "l"(src + off), "r"(nb), "r"(smem_u32(&full[s]))
        : "memory");
  };
  for (int c = 0; c < NS - 1 && c < nchunks; ++c) issue(c);
  for (int c = 0; c < nchunks; ++c) {
    int s = c % NS;
    uint32_t parity = (c / NS) & 1;
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(smem_u32(&full[s])), "r"(parity)
          : "memory");
    }
    size_t off = lo + (size_t)c * chunk;
    uint32_t nb = (uint32_t)((hi - off) < (size_t)chunk ? (hi - off) : chunk);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off),
                 "r"(smem_u32(smem + (size_t)s * chunk)), "r"(nb)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // the stage refilled next is (c + NS - 1) % NS == (c - 1) % NS: its store
    // (issued one iteration ago) must have finished reading shared memory
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    if (c + NS - 1 < nchunks) issue(c + NS - 1);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  size_t bytes = (argc > 1 ? atoll(argv[1]) : 256) << 20;
  int ndev;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("need 2 GPUs\n");
    return 1;
  }
  float* buf[2][2];  // [dev][src/dst]
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&buf[d][0], bytes));
    CK(cudaMalloc(&buf[d][1], bytes));
    CK(cudaMemset(buf[d][0], 1, bytes));
  }
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaStreamCreate(&st[d]));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  auto run = [&](const char* name, int both, auto launch) {
    for (int rep = 0; rep < 4; ++rep) {
      for (int d = 0; d < 2; ++d) {
        if (!both && d == 0) continue;
        CK(cudaSetDevice(d));
        CK(cudaEventRecord(e0[d], st[d]));
        launch(d, st[d], buf[1 - d][0], buf[d][1]);
        CK(cudaEventRecord(e1[d], st[d]));
      }
      float ms = 0;
      for (int d = 0; d < 2; ++d) {
        if (!both && d == 0) continue;
        CK(cudaSetDevice(d));
        CK(cudaEventSynchronize(e1[d]));
        float t;
        CK(cudaEventElapsedTime(&t, e0[d], e1[d]));
        ms = t > ms ? t : ms;
      }
      if (rep == 3)
        printf("%-28s %s  %8.1f GB/s per GPU  (%.3f ms)\n", name, both ? "bidir " : "1-way ",
               bytes / ms / 1e6, ms);
    }
  };
  for (int both = 0; both < 2; ++both) {
    run("ldg U=2 148x512", both, [&](int d, cudaStream_t s, float* src, float* dst) {
      ldg_copy<2><<<148, 512, 0, s>>>((const float4*)src, (float4*)dst, bytes / 16);
    });
    run("ldg U=8 148x512", both, [&](int d, cudaStream_t s, float* src, float* dst) {
      ldg_copy<8><<<148, 512, 0, s>>>((const float4*)src, (float4*)dst, bytes / 16);
    });
    run("ldg U=8 296x512", both, [&](int d, cudaStream_t s, float* src, float* dst) {
      ldg_copy<8><<<296, 512, 0, s>>>((const float4*)src, (float4*)dst, bytes / 16);
    });
    for (int chunk : {8192, 16384, 32768}) {
      for (int ctas : {148, 296}) {
        char nm[64];
        snprintf(nm, sizeof nm, "bulk NS=4 %dKB %dcta", chunk / 1024, ctas);
        run(nm, both, [&](int d, cudaStream_t s, float* src, float* dst) {
          CK(cudaFuncSetAttribute(bulk_copy<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  4 * chunk));
          bulk_copy<4><<<ctas, 128, 4 * chunk, s>>>((const char*)src, (char*)dst, bytes, chunk);
        });
      }
    }
    run("cudaMemcpyPeerAsync", both, [&](int d, cudaStream_t s, float* src, float* dst) {
      CK(cudaMemcpyPeerAsync(dst, d, src, 1 - d, bytes, s));
    });
    // push: this GPU reads its own HBM and stores into the peer's buffer
    run("push stg U=2 148x512", both, [&](int d, cudaStream_t s, float* src, float* dst) {
      ldg_copy<2><<<148, 512, 0, s>>>((const float4*)buf[d][0], (float4*)buf[1 - d][1],
                                      bytes / 16);
    });
    run("push stg U=4 296x512", both, [&](int d, cudaStream_t s, float* src, float* dst) {
      ldg_copy<4><<<296, 512, 0, s>>>((const float4*)buf[d][0], (float4*)buf[1 - d][1],
                                      bytes / 16);
    });
    for (int chunk : {16384, 32768}) {
      char nm[64];
      snprintf(nm, sizeof nm, "push bulk NS=4 %dKB 148cta", chunk / 1024);
      run(nm, both, [&](int d, cudaStream_t s, float* src, float* dst) {
        CK(cudaFuncSetAttribute(bulk_copy<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                4 * chunk));
        bulk_copy<4><<<148, 128, 4 * chunk, s>>>((const char*)buf[d][0], (char*)buf[1 - d][1],
                                                 bytes, chunk);
      });
    }
  }
  // correctness of the bulk path
  CK(cudaSetDevice(1));
  CK(cudaMemset(buf[1][1], 0, bytes));
  bulk_copy<4><<<148, 128, 4 * 16384, st[1]>>>((const char*)buf[0][0], (char*)buf[1][1], bytes,
                                               16384);
  CK(cudaStreamSynchronize(st[1]));
  unsigned char* h = (unsigned char*)malloc(bytes);
  CK(cudaMemcpy(h, buf[1][1], bytes, cudaMemcpyDeviceToHost));
  size_t bad = 0;
  for (size_t i = 0; i < bytes; ++i) bad += h[i] != 1;
  printf("bulk copy correctness: %zu bad bytes\n", bad);
  return 0;
}
