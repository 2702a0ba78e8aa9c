// The reference's gradient producer on the device: ToyModel.loss_and_grad_sum
// (/root/reference/pkg/src/minidist/sgd.py:220-248) for every worker of a
// node, writing node_gradient's per-worker buffer (sgd.py:335-353):
// [float32 gradient sum | loss sum | correct count].
//
// One CTA per worker sub-batch; the batch is the DIMD minibatch slots
// (records = little-endian float32 features, sgd.py:310-313; float64
// features for the reference's ``grad(model, batch)`` API, sgd.py:250-257). The math is
// float64 from the float32 weights, rounded to float32 once at the end, in
// the reference's (numpy's) evaluation order:
//   * every matmul output element accumulates over its inner index in order
//     with fused multiply-adds (OpenBLAS dgemm's order, measured against
//     numpy in the build container);
//   * softmax row sums sequential, column sums (axis 0) sequential over rows,
//     the loss sum numpy's pairwise summation;
//   * argmax = first maximum; labels wrap like numpy indices (y < 0 -> y + C).
// Tiny (the reference's model has 172 parameters): latency-bound, one launch
// per step for all workers.
#include <cuda_runtime.h>

#include "md_common.cuh"

namespace md {

namespace {

constexpr int kToyThreads = 256;

struct ToyArgs {
  const float* w;
  int32_t n_in, hidden, ncls, batch;
  int32_t feature_bytes;  // 4: float32 records (the DIMD format), 8: float64 features
  int64_t record_stride;
  const uint8_t* records[MD_MAX_WORKERS];
  const int32_t* labels[MD_MAX_WORKERS];
  float* out[MD_MAX_WORKERS];
  int32_t* status;  // nullable: 1 + a row whose label is out of range (the first to report)
};

// numpy's pairwise_sum (umath/loops_utils.h.src) over n float64 values
__device__ double np_pairwise(const double* a, int n) {
  if (n < 8) {
    double r = -0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise(a, n2), np_pairwise(a + n2, n - n2));
}

__global__ void __launch_bounds__(kToyThreads) toy_grad_kernel(const __grid_constant__ ToyArgs a) {
  extern __shared__ __align__(16) double sm[];
  const int k = a.batch, n_in = a.n_in, H = a.hidden, C = a.ncls;
  const int o_b1 = n_in * H, o_w2 = o_b1 + H, o_b2 = o_w2 + H * C, p = o_b2 + C;
  double* w = sm;             // [p]
  double* x = w + p;          // [k][n_in]
  double* h = x + k * n_in;   // [k][H]
  double* pr = h + k * H;     // [k][C]: z, then p, then dz
  double* da = pr + k * C;    // [k][H]
  double* lt = da + k * H;    // [k]: -log p[y]
  int* lab = reinterpret_cast<int*>(lt + k);  // [k]
  __shared__ int s_correct;
  const int wk = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const uint8_t* rec = a.records[wk];
  const int32_t* labels = a.labels[wk];
  float* out = a.out[wk];

  if (tid == 0) s_correct = 0;
  for (int i = tid; i < p; i += nt) w[i] = static_cast<double>(a.w[i]);
  for (int e = tid; e < k * n_in; e += nt) {
    const int r = e / n_in, i = e % n_in;
    const uint8_t* b = rec + r * a.record_stride + a.feature_bytes * i;
    uint64_t bits = 0;
    for (int q = a.feature_bytes - 1; q >= 0; --q) bits = (bits << 8) | b[q];  // little endian
    x[e] = a.feature_bytes == 8 ? __longlong_as_double(static_cast<long long>(bits))
                                : static_cast<double>(__uint_as_float(static_cast<uint32_t>(bits)));
  }
  for (int r = tid; r < k; r += nt) {
    int y = labels[r];
    if (y < 0) y += C;  // numpy fancy index
    if (y < 0 || y >= C) {
      if (a.status) atomicCAS(a.status, 0, r + 1);
      y = 0;
    }
    lab[r] = y;
  }
  __syncthreads();

  // h = tanh(x @ W1 + b1)
  for (int e = tid; e < k * H; e += nt) {
    const int r = e / H, j = e % H;
    double acc = 0.0;
    for (int i = 0; i < n_in; ++i) acc = fma(x[r * n_in + i], w[i * H + j], acc);
    h[e] = tanh(__dadd_rn(acc, w[o_b1 + j]));
  }
  __syncthreads();

  // per row: z = h @ W2 + b2, softmax, -log p[y], argmax, dz = p - onehot(y)
  for (int r = tid; r < k; r += nt) {
    double* z = pr + r * C;
    double zmax = -INFINITY;
    for (int c = 0; c < C; ++c) {
      double acc = 0.0;
      for (int j = 0; j < H; ++j) acc = fma(h[r * H + j], w[o_w2 + j * C + c], acc);
      z[c] = __dadd_rn(acc, w[o_b2 + c]);
      zmax = fmax(zmax, z[c]);
    }
    double s = -0.0;
    int arg = 0;
    for (int c = 0; c < C; ++c) {
      z[c] = __dsub_rn(z[c], zmax);
      if (z[c] > z[arg]) arg = c;
    }
    for (int c = 0; c < C; ++c) {
      z[c] = exp(z[c]);
      s = __dadd_rn(s, z[c]);
    }
    for (int c = 0; c < C; ++c) z[c] = __ddiv_rn(z[c], s);
    const int y = lab[r];
    lt[r] = -log(z[y]);
    if (arg == y) atomicAdd(&s_correct, 1);
    z[y] = __dsub_rn(z[y], 1.0);
  }
  __syncthreads();

  // da = (1 - h*h) * (dz @ W2.T); the loss sum on the last warp's lane 0
  if (tid == nt - 1) out[p] = __double2float_rn(__dadd_rn(0.0, np_pairwise(lt, k)));
  for (int e = tid; e < k * H; e += nt) {
    const int r = e / H, j = e % H;
    double acc = 0.0;
    for (int c = 0; c < C; ++c) acc = fma(pr[r * C + c], w[o_w2 + j * C + c], acc);
    const double hv = h[e];
    da[e] = __dmul_rn(__dsub_rn(1.0, __dmul_rn(hv, hv)), acc);
  }
  __syncthreads();

  // dW1 = x.T @ da, db1 = da.sum(0), dW2 = h.T @ dz, db2 = dz.sum(0)
  for (int e = tid; e < p; e += nt) {
    double acc = 0.0;
    if (e < o_b1) {
      const int i = e / H, j = e % H;
      for (int r = 0; r < k; ++r) acc = fma(x[r * n_in + i], da[r * H + j], acc);
    } else if (e < o_w2) {
      const int j = e - o_b1;
      for (int r = 0; r < k; ++r) acc = __dadd_rn(acc, da[r * H + j]);
    } else if (e < o_b2) {
      const int j = (e - o_w2) / C, c = (e - o_w2) % C;
      for (int r = 0; r < k; ++r) acc = fma(h[r * H + j], pr[r * C + c], acc);
    } else {
      const int c = e - o_b2;
      for (int r = 0; r < k; ++r) acc = __dadd_rn(acc, pr[r * C + c]);
    }
    out[e] = __double2float_rn(acc);
  }
  if (tid == 0) out[p + 1] = static_cast<float>(s_correct);
}

size_t toy_smem_bytes(int64_t k, int64_t n_in, int64_t H, int64_t C) {
  const int64_t p = n_in * H + H + H * C + C;
  return static_cast<size_t>(8 * (p + k * (n_in + 2 * H + C) + k) + 4 * k);
}

}  // namespace

}  // namespace md

extern "C" int md_toy_grad(const float* w, int32_t n_in, int32_t hidden, int32_t n_classes,
                           const uint8_t* const* records, int32_t feature_bytes,
                           const int32_t* const* labels, int64_t record_stride, int32_t batch,
                           float* const* out, int32_t n_workers, int32_t* status, void* stream) {
  if (!w || !records || !labels || !out || n_in < 1 || hidden < 1 || n_classes < 1 ||
      batch < 1 || n_workers < 1) {
    md::set_error("md_toy_grad: null pointer or non-positive size");
    return MD_ERR_INVALID_CONFIG;
  }
  if (feature_bytes != 4 && feature_bytes != 8) {
    md::set_error("md_toy_grad: feature_bytes must be 4 or 8, got %d", feature_bytes);
    return MD_ERR_INVALID_CONFIG;
  }
  if (record_stride < static_cast<int64_t>(feature_bytes) * n_in) {
    md::set_error("md_toy_grad: records of %lld bytes hold fewer than %d features",
                  static_cast<long long>(record_stride), n_in);
    return MD_ERR_LENGTH_MISMATCH;
  }
  const size_t smem = md::toy_smem_bytes(batch, n_in, hidden, n_classes);
  static std::atomic<uint64_t> attr_done{0};
  int dev = 0;
  MD_CUDA_TRY(cudaGetDevice(&dev));
  int optin = 0;
  MD_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  cudaFuncAttributes fa{};
  MD_CUDA_TRY(cudaFuncGetAttributes(&fa, md::toy_grad_kernel));
  optin -= static_cast<int>(fa.sharedSizeBytes);  // the kernel's static shared memory
  if (smem > static_cast<size_t>(optin)) {
    md::set_error("md_toy_grad: batch %d x (%d in, %d hidden, %d classes) needs %zu B of shared "
                  "memory (> %d)", batch, n_in, hidden, n_classes, smem, optin);
    return MD_ERR_INVALID_CONFIG;
  }
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_done.load() & bit)) {
    MD_CUDA_TRY(cudaFuncSetAttribute(md::toy_grad_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
    attr_done.fetch_or(bit);
  }
  for (int32_t w0 = 0; w0 < n_workers; w0 += MD_MAX_WORKERS) {
    md::ToyArgs a{};
    a.w = w;
    a.n_in = n_in;
    a.hidden = hidden;
    a.ncls = n_classes;
    a.batch = batch;
    a.feature_bytes = feature_bytes;
    a.record_stride = record_stride;
    a.status = status;
    const int m = std::min<int32_t>(MD_MAX_WORKERS, n_workers - w0);
    for (int j = 0; j < m; ++j) {
      a.records[j] = records[w0 + j];
      a.labels[j] = labels[w0 + j];
      a.out[j] = out[w0 + j];
      if (!a.records[j] || !a.labels[j] || !a.out[j]) {
        md::set_error("md_toy_grad: null buffer for worker %d", w0 + j);
        return MD_ERR_INVALID_CONFIG;
      }
    }
    md::toy_grad_kernel<<<m, md::kToyThreads, smem, md::as_stream(stream)>>>(a);
    MD_LAUNCH_CHECK();
  }
  return MD_OK;
}
