// nvls_probe: is NVLS multicast (multimem.st through the NVSwitch) a faster
// broadcast leg than unicast pushes for the owner-push allreduce?
//
// One process drives N GPUs (N = all visible, 2..8). A multicast object of
// `bytes` is bound to one physical allocation per GPU. The all-gather
// pattern of the broadcast leg: GPU j holds slice j (bytes / N) and must
// deliver it to every GPU.
//   unicast   GPU j stores its slice into every peer's buffer (P2P, float4
//             stores through NVLink) -- what allreduce_push_kernel does
//             (there with TMA bulk stores);
//   multicast GPU j stores its slice ONCE to the multicast address
//             (multimem.st.relaxed.sys.global.v4.f32); the switch replicates
//             it into every bound GPU, the writer included.
// All GPUs run concurrently; time = max over GPUs (events), median of reps.
// Each buffer is then checked: every slice must hold its owner's pattern.
// Also: multimem.ld_reduce.add.f32 at N = 2 vs the plain f32 sum (bitwise).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvls_probe tools/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));              \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)
#define CU(x)                                                                              \
  do {                                                                                     \
    CUresult r = (x);                                                                      \
    if (r != CUDA_SUCCESS) {                                                               \
      const char* s = nullptr;                                                             \
      cuGetErrorString(r, &s);                                                             \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, s ? s : "?");                        \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

__global__ void __launch_bounds__(512) fill_slice(float4* dst, size_t n4, float tag) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = make_float4(tag, tag + 1.f, tag + 2.f, (float)(i & 1023));
}

// slice [lo, lo + n4) of src -> the same range of every destination
template <int U>
__global__ void __launch_bounds__(512) unicast_push(const float4* __restrict__ src, float4** dsts,
                                                    int ndst, size_t n4) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t b = blockIdx.x * (size_t)blockDim.x * U + threadIdx.x; b < n4; b += stride) {
    float4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (b + (size_t)u * blockDim.x < n4) x[u] = __ldcs(src + b + (size_t)u * blockDim.x);
    for (int d = 0; d < ndst; ++d)
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (b + (size_t)u * blockDim.x < n4) dsts[d][b + (size_t)u * blockDim.x] = x[u];
  }
}

template <int U>
__global__ void __launch_bounds__(512) multicast_push(const float4* __restrict__ src, float4* mc,
                                                      size_t n4) {
  const size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t b = blockIdx.x * (size_t)blockDim.x * U + threadIdx.x; b < n4; b += stride) {
    float4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (b + (size_t)u * blockDim.x < n4) x[u] = __ldcs(src + b + (size_t)u * blockDim.x);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (b + (size_t)u * blockDim.x < n4) {
        float4* p = mc + b + (size_t)u * blockDim.x;
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p),
                     "f"(x[u].x), "f"(x[u].y), "f"(x[u].z), "f"(x[u].w)
                     : "memory");
      }
  }
}

__global__ void __launch_bounds__(512) mc_reduce(const float4* mc, float4* out, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
       i += (size_t)gridDim.x * blockDim.x) {
    float4 r;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(mc + i)
                 : "memory");
    out[i] = r;
  }
}

__global__ void check_slices(const float4* buf, size_t n4, int N, unsigned long long* bad) {
  const size_t per = n4 / N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per * N;
       i += (size_t)gridDim.x * blockDim.x) {
    const int owner = (int)(i / per);
    const size_t k = i - (size_t)owner * per;
    const float tag = 10.f * owner + 1.f;
    float4 x = buf[i];
    if (x.x != tag || x.y != tag + 1.f || x.z != tag + 2.f || x.w != (float)(k & 1023))
      atomicAdd(bad, 1ull);
  }
}

int main(int argc, char** argv) {
  size_t mb = argc > 1 ? atoll(argv[1]) : 256;
  int reps = argc > 2 ? atoi(argv[2]) : 10;
  CU(cuInit(0));
  int N = 0;
  CK(cudaGetDeviceCount(&N));
  if (N < 2) {
    printf("need >= 2 GPUs\n");
    return 0;
  }
  int mcs = 0;
  CUdevice d0;
  CU(cuDeviceGet(&d0, 0));
  CU(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d0));
  printf("N=%d multicast_supported=%d\n", N, mcs);
  if (!mcs) return 0;
  for (int a = 0; a < N; ++a)
    for (int b = 0; b < N; ++b)
      if (a != b) {
        CK(cudaSetDevice(a));
        cudaDeviceEnablePeerAccess(b, 0);
        cudaGetLastError();
      }
  CUmulticastObjectProp prop = {};
  prop.numDevices = N;
  prop.handleTypes = 0;
  size_t gran = 0;
  prop.size = mb << 20;
  CU(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  size_t bytes = ((mb << 20) + gran - 1) / gran * gran;
  bytes = bytes / (16 * N * gran) * (16 * N * gran);
  if (bytes == 0) bytes = 16 * N * gran;
  prop.size = bytes;
  CUmemGenericAllocationHandle mc;
  CU(cuMulticastCreate(&mc, &prop));
  for (int d = 0; d < N; ++d) {
    CUdevice dev;
    CU(cuDeviceGet(&dev, d));
    CU(cuMulticastAddDevice(mc, dev));
  }
  std::vector<float4*> uva(N), mcva(N), src(N), out(N);
  std::vector<CUmemGenericAllocationHandle> phys(N);
  for (int d = 0; d < N; ++d) {
    CK(cudaSetDevice(d));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    size_t pg = 0;
    CU(cuMemGetAllocationGranularity(&pg, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    CU(cuMemCreate(&phys[d], bytes, &ap, 0));
    CU(cuMulticastBindMem(mc, 0, phys[d], 0, bytes, 0));
    CUdeviceptr p;
    CU(cuMemAddressReserve(&p, bytes, gran, 0, 0));
    CU(cuMemMap(p, bytes, 0, phys[d], 0));
    std::vector<CUmemAccessDesc> acc(N);
    for (int e = 0; e < N; ++e) {
      acc[e].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      acc[e].location.id = e;
      acc[e].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    }
    CU(cuMemSetAccess(p, bytes, acc.data(), N));
    uva[d] = reinterpret_cast<float4*>(p);
    CUdeviceptr q;
    CU(cuMemAddressReserve(&q, bytes, gran, 0, 0));
    CU(cuMemMap(q, bytes, 0, mc, 0));
    CUmemAccessDesc a1 = {};
    a1.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    a1.location.id = d;
    a1.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU(cuMemSetAccess(q, bytes, &a1, 1));
    mcva[d] = reinterpret_cast<float4*>(q);
    CK(cudaMalloc(&src[d], bytes / N));
    CK(cudaMalloc(&out[d], bytes));
    fill_slice<<<592, 512>>>(src[d], bytes / N / 16, 10.f * d + 1.f);
    CK(cudaDeviceSynchronize());
  }
  const size_t n4 = bytes / N / 16;  // float4 per slice
  printf("buffer %zu MB (granularity %zu KB), slice %zu MB per GPU\n", bytes >> 20, gran >> 10,
         (bytes / N) >> 20);
  std::vector<cudaStream_t> st(N);
  std::vector<cudaEvent_t> e0(N), e1(N);
  std::vector<float4**> dsts(N);
  for (int d = 0; d < N; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
    std::vector<float4*> h(N);
    for (int e = 0; e < N; ++e) h[e] = uva[(d + 1 + e) % N] + (size_t)d * n4;  // peers first
    CK(cudaMalloc(&dsts[d], N * sizeof(float4*)));
    CK(cudaMemcpy(dsts[d], h.data(), N * sizeof(float4*), cudaMemcpyHostToDevice));
  }
  unsigned long long* bad;
  CK(cudaMallocManaged(&bad, sizeof(*bad)));
  for (int mode = 0; mode < 2; ++mode) {
    for (int grid : {148, 296, 592}) {
      std::vector<float> ms;
      for (int r = 0; r < reps + 2; ++r) {
        for (int d = 0; d < N; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaMemsetAsync(uva[d], 0, bytes, st[d]));
        }
        for (int d = 0; d < N; ++d) CK(cudaStreamSynchronize(st[d]));
        for (int d = 0; d < N; ++d) {
          CK(cudaSetDevice(d));
          CK(cudaEventRecord(e0[d], st[d]));
          if (mode == 0)
            unicast_push<4><<<grid, 512, 0, st[d]>>>(src[d], dsts[d], N, n4);
          else
            multicast_push<4><<<grid, 512, 0, st[d]>>>(src[d], mcva[d] + (size_t)d * n4, n4);
          CK(cudaEventRecord(e1[d], st[d]));
        }
        float mx = 0.f;
        for (int d = 0; d < N; ++d) {
          CK(cudaEventSynchronize(e1[d]));
          float t;
          CK(cudaEventElapsedTime(&t, e0[d], e1[d]));
          mx = std::max(mx, t);
        }
        if (r >= 2) ms.push_back(mx);
      }
      std::sort(ms.begin(), ms.end());
      const float med = ms[ms.size() / 2];
      *bad = 0;
      for (int d = 0; d < N; ++d) {
        CK(cudaSetDevice(d));
        check_slices<<<592, 512>>>(uva[d], n4 * N, N, bad);
        CK(cudaDeviceSynchronize());
      }
      // per GPU: ingress (N-1)/N of the buffer in both modes (multicast also
      // re-delivers the own slice through the switch); "algbw" = bytes / t
      const double gb = (double)bytes * (N - 1) / N / (med * 1e-3) / 1e9;
      printf("%-10s grid %4d: %8.3f ms  %7.1f GB/s per GPU (peer bytes in)  bad=%llu\n",
             mode ? "multicast" : "unicast", grid, med, gb, *bad);
    }
  }
  if (N == 2) {  // in-switch reduction: bitwise vs the plain f32 add?
    for (int d = 0; d < N; ++d) {
      CK(cudaSetDevice(d));
      fill_slice<<<592, 512>>>(uva[d], bytes / 16, 0.1f + 0.37f * d);
      CK(cudaDeviceSynchronize());
    }
    CK(cudaSetDevice(0));
    mc_reduce<<<592, 512>>>(mcva[0], out[0], bytes / 16);
    CK(cudaDeviceSynchronize());
    std::vector<float> a(bytes / 4), b(bytes / 4), o(bytes / 4);
    CK(cudaMemcpy(a.data(), uva[0], bytes, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), uva[1], bytes, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(o.data(), out[0], bytes, cudaMemcpyDeviceToHost));
    size_t diff = 0;
    for (size_t i = 0; i < a.size(); ++i) {
      float s = a[i] + b[i];
      if (memcmp(&s, &o[i], 4) != 0) ++diff;
    }
    printf("multimem.ld_reduce.add.f32 at N=2: %zu of %zu words differ from a+b\n", diff, a.size());
  }
  return 0;
}
