// gather_variants: record gather (DIMD random_batch) kernel variants on a
// C4-sized shard (160,000 x 150,528 B = 24 GB) with 8,192 random picks --
// which loop shape gets closest to the HBM copy peak?
//   A  (record, 32 KB chunk) units, 512 thr, 4 x 16 B per thread, 4 CTA/SM (md::gather_kernel)
//   B  same units, 8 x 16 B per thread in flight (loads of two units overlapped)
//   C  (record, 64 KB chunk) units, 512 thr, 8 x 16 B per thread
//   D  (record, 16 KB chunk) units, 256 thr, 4 x 16 B per thread, 8 CTA/SM
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_variants tools/gather_variants.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));     \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

constexpr uint64_t REC = 224 * 224 * 3;

template <int U, int CHUNK>
__global__ void gather_units(const uint8_t* blob, const uint64_t* off, const int64_t* picks,
                             int64_t batch, uint8_t* out) {
  const int chunks = (REC + CHUNK - 1) / CHUNK;
  const int64_t units = batch * chunks;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t b = u / chunks;
    const int c = static_cast<int>(u % chunks);
    const uint64_t lo = static_cast<uint64_t>(c) * CHUNK;
    const uint64_t n = min(static_cast<uint64_t>(CHUNK), REC - lo);
    const uint4* s4 = reinterpret_cast<const uint4*>(blob + off[picks[b]] + lo);
    uint4* d4 = reinterpret_cast<uint4*>(out + b * REC + lo);
    const uint64_t nv = n / 16;
    for (uint64_t k0 = threadIdx.x; k0 < nv; k0 += static_cast<uint64_t>(blockDim.x) * U) {
      uint4 x[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const uint64_t k = k0 + static_cast<uint64_t>(q) * blockDim.x;
        if (k < nv) x[q] = __ldcs(s4 + k);
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const uint64_t k = k0 + static_cast<uint64_t>(q) * blockDim.x;
        if (k < nv) __stcs(d4 + k, x[q]);
      }
    }
  }
}

// B: two units per CTA iteration, all loads of both issued before any store
__global__ void gather_pairs(const uint8_t* blob, const uint64_t* off, const int64_t* picks,
                             int64_t batch, uint8_t* out) {
  constexpr int CHUNK = 32768, U = 4;
  const int chunks = (REC + CHUNK - 1) / CHUNK;
  const int64_t units = batch * chunks;
  for (int64_t u = 2 * static_cast<int64_t>(blockIdx.x); u < units; u += 2 * gridDim.x) {
    uint4 x[2][U];
    const uint4* s[2];
    uint4* d[2];
    uint64_t nv[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t uu = u + h;
      nv[h] = 0;
      if (uu < units) {
        const int64_t b = uu / chunks;
        const int c = static_cast<int>(uu % chunks);
        const uint64_t lo = static_cast<uint64_t>(c) * CHUNK;
        nv[h] = min(static_cast<uint64_t>(CHUNK), REC - lo) / 16;
        s[h] = reinterpret_cast<const uint4*>(blob + off[picks[b]] + lo);
        d[h] = reinterpret_cast<uint4*>(out + b * REC + lo);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const uint64_t k = threadIdx.x + static_cast<uint64_t>(q) * blockDim.x;
        if (k < nv[h]) x[h][q] = __ldcs(s[h] + k);
      }
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const uint64_t k = threadIdx.x + static_cast<uint64_t>(q) * blockDim.x;
        if (k < nv[h]) __stcs(d[h] + k, x[h][q]);
      }
  }
}

namespace libcopy {
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

constexpr uint64_t kGatherChunk = 32 * 1024;

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
}  // namespace libcopy

int main() {
  const int64_t n_rec = 160000, batch = 8192;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint8_t *blob, *out;
  uint64_t* off;
  int64_t* picks;
  CK(cudaMalloc(&blob, n_rec * REC));
  CK(cudaMemset(blob, 1, n_rec * REC));
  CK(cudaMalloc(&out, batch * REC));
  std::vector<uint64_t> h_off(n_rec);
  for (int64_t i = 0; i < n_rec; ++i) h_off[i] = i * REC;
  CK(cudaMalloc(&off, n_rec * 8));
  CK(cudaMemcpy(off, h_off.data(), n_rec * 8, cudaMemcpyHostToDevice));
  std::vector<int64_t> h_p(batch);
  uint64_t st = 12345;
  for (auto& p : h_p) {
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    p = static_cast<int64_t>((st >> 33) % n_rec);
  }
  CK(cudaMalloc(&picks, batch * 8));
  CK(cudaMemcpy(picks, h_p.data(), batch * 8, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    std::vector<float> ms;
    for (int r = 0; r < 9; ++r) {
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float t;
      CK(cudaEventElapsedTime(&t, e0, e1));
      ms.push_back(t);
    }
    std::sort(ms.begin(), ms.end());
    const double gb = 2.0 * batch * REC / (ms[4] * 1e-3) / 1e9;
    printf("%-44s %7.3f ms  %7.1f GB/s (read+write)\n", name, ms[4], gb);
  };
  run("A 32KB units, 512thr, U4, 4 CTA/SM", [&] {
    gather_units<4, 32768><<<sms * 4, 512>>>(blob, off, picks, batch, out);
  });
  run("A' same, 8 CTA/SM (grid)", [&] {
    gather_units<4, 32768><<<sms * 8, 512>>>(blob, off, picks, batch, out);
  });
  run("B 32KB unit pairs, 512thr, U4 x 2", [&] {
    gather_pairs<<<sms * 4, 512>>>(blob, off, picks, batch, out);
  });
  run("C 64KB units, 512thr, U8", [&] {
    gather_units<8, 65536><<<sms * 4, 512>>>(blob, off, picks, batch, out);
  });
  run("D 16KB units, 256thr, U4, 8 CTA/SM", [&] {
    gather_units<4, 16384><<<sms * 8, 256>>>(blob, off, picks, batch, out);
  });
  run("E whole records, 1024thr, U8", [&] {
    gather_units<8, 151552><<<sms * 2, 1024>>>(blob, off, picks, batch, out);
  });
  uint32_t *len, *label, *olab;
  int32_t* bad;
  {
    std::vector<uint32_t> h_len(n_rec, static_cast<uint32_t>(REC));
    CK(cudaMalloc(&len, n_rec * 4));
    CK(cudaMemcpy(len, h_len.data(), n_rec * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&label, n_rec * 4));
    CK(cudaMemset(label, 0, n_rec * 4));
    CK(cudaMalloc(&olab, batch * 4));
    CK(cudaMalloc(&bad, 4));
    CK(cudaMemset(bad, 0, 4));
  }
  const int chunks = (REC + 32768 - 1) / 32768;
  run("L library gather_kernel, grid 4/SM", [&] {
    libcopy::gather_kernel<<<sms * 4, 512>>>(blob, off, len, label, picks, batch, out, REC, nullptr,
                                             olab, bad, chunks);
  });
  run("L library gather_kernel, grid 8/SM", [&] {
    libcopy::gather_kernel<<<sms * 8, 512>>>(blob, off, len, label, picks, batch, out, REC, nullptr,
                                             olab, bad, chunks);
  });
  CK(cudaFuncSetAttribute(libcopy::gather_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                          cudaSharedmemCarveoutMaxShared));
  run("L library gather_kernel, 8/SM, max-shared carveout", [&] {
    libcopy::gather_kernel<<<sms * 8, 512>>>(blob, off, len, label, picks, batch, out, REC, nullptr,
                                             olab, bad, chunks);
  });
  run("copy: cudaMemcpy D2D of the same bytes", [&] {
    CK(cudaMemcpyAsync(out, blob, batch * REC, cudaMemcpyDeviceToDevice));
  });
  return 0;
}
