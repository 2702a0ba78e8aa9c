// The reference's gradient producer on the device: ToyModel.loss_and_grad_sum
// (/root/reference/pkg/src/minidist/sgd.py:220-248) for every worker of a
// node, writing node_gradient's per-worker buffer (sgd.py:335-353):
// [float32 gradient sum | loss sum | correct count].
//
// Inputs are the DIMD minibatch slots (records = little-endian float32
// features, sgd.py:310-313; float64 features for the reference's
// ``grad(model, batch)`` API, sgd.py:250-257). The math is float64 from the
// float32 weights, rounded to float32 once at the end, in the reference's
// (numpy's) evaluation order:
//   * every matmul output element accumulates over its inner index in order
//     with fused multiply-adds (OpenBLAS dgemm's order, measured against
//     numpy in the build container);
//   * softmax row sums sequential, column sums (axis 0) sequential over rows,
//     the loss sum numpy's pairwise summation;
//   * argmax = first maximum; labels wrap like numpy indices (y < 0 -> y + C).
// Six small launches per step, parallel over (worker, output element): input
// conversion, hidden layer, logits (one CTA per row, operands staged in shared
// memory), softmax rows, hidden gradient, parameter gradients.
// Intermediates live in a caller-provided float64 workspace, so any model
// size works (the reference's bench_train default is 16 -> 2048 -> 4).
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
  int64_t work_stride;    // doubles of workspace per worker
  double* work;           // [worker][x | h | z/p/dz | da | lt | lab | correct]
  const uint8_t* records[MD_MAX_WORKERS];
  const int32_t* labels[MD_MAX_WORKERS];
  float* out[MD_MAX_WORKERS];
  int32_t* status;  // nullable: 1 + a row whose label is out of range (the first to report)
};

struct Work {
  double *x, *h, *pr, *da, *lt;
  int* lab;
  int* correct;
};

__device__ __forceinline__ Work work_of(const ToyArgs& a, int wk) {
  const int64_t k = a.batch, H = a.hidden, C = a.ncls;
  double* b = a.work + wk * a.work_stride;
  Work w;
  w.x = b;                 // [k][n_in]: the features as float64
  w.h = w.x + k * a.n_in;  // [k][H]
  w.pr = w.h + k * H;      // [k][C]: z, then p, then dz
  w.da = w.pr + k * C;     // [k][H]
  w.lt = w.da + k * H;     // [k]: -log p[y]
  w.lab = reinterpret_cast<int*>(w.lt + k);  // [k]
  w.correct = w.lab + k;   // [1]
  return w;
}

int64_t work_doubles(int64_t k, int64_t n_in, int64_t H, int64_t C) {
  return k * (n_in + 2 * H + C + 1) + (k + 2 + 1) / 2;
}

// feature i of row r, as float64 (little endian; the records are byte rows)
__device__ __forceinline__ double feat(const ToyArgs& a, const uint8_t* rec, int64_t r, int i) {
  const uint8_t* b = rec + r * a.record_stride + static_cast<int64_t>(a.feature_bytes) * i;
  if (a.feature_bytes == 4) {
    if ((reinterpret_cast<uintptr_t>(b) & 3) == 0)
      return static_cast<double>(__ldg(reinterpret_cast<const float*>(b)));
    const uint32_t bits = b[0] | (b[1] << 8) | (b[2] << 16) | (static_cast<uint32_t>(b[3]) << 24);
    return static_cast<double>(__uint_as_float(bits));
  }
  if ((reinterpret_cast<uintptr_t>(b) & 7) == 0) return __ldg(reinterpret_cast<const double*>(b));
  uint64_t bits = 0;
  for (int q = 7; q >= 0; --q) bits = (bits << 8) | b[q];
  return __longlong_as_double(static_cast<long long>(bits));
}

__device__ __forceinline__ double wv(const ToyArgs& a, int64_t i) {
  return static_cast<double>(__ldg(a.w + i));
}

// numpy's pairwise_sum (umath/loops_utils.h.src) over n float64 values
__device__ double np_pairwise(const double* v, int64_t n) {
  if (n < 8) {
    double r = -0.0;
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, v[i]);
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = v[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], v[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, v[i]);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise(v, n2), np_pairwise(v + n2, n - n2));
}

// grid: (blocks per worker, workers); e strides over one worker's elements
#define TOY_LOOP(e, count)                                                          \
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; \
       e < (count); e += static_cast<int64_t>(gridDim.x) * blockDim.x)

// 1. features as float64, labels
__global__ void __launch_bounds__(kToyThreads) toy_input_kernel(const __grid_constant__ ToyArgs a) {
  const int wk = blockIdx.y;
  const Work w = work_of(a, wk);
  const int k = a.batch, n_in = a.n_in, C = a.ncls;
  const uint8_t* rec = a.records[wk];
  TOY_LOOP(e, static_cast<int64_t>(k) * n_in) {
    w.x[e] = feat(a, rec, e / n_in, static_cast<int>(e % n_in));
  }
  TOY_LOOP(r, k) {
    int y = a.labels[wk][r];
    if (y < 0) y += C;  // numpy fancy index
    if (y < 0 || y >= C) {
      if (a.status) atomicCAS(a.status, 0, static_cast<int>(r) + 1);
      y = 0;
    }
    w.lab[r] = y;
    if (r == 0) *w.correct = 0;
  }
}

// 2. h = tanh(x @ W1 + b1); the loads of a chain do not depend on it, so the
// unrolled loop keeps them in flight ahead of the fused multiply-adds
__global__ void __launch_bounds__(kToyThreads) toy_hidden_kernel(const __grid_constant__ ToyArgs a) {
  const Work w = work_of(a, blockIdx.y);
  const int k = a.batch, n_in = a.n_in, H = a.hidden;
  TOY_LOOP(e, static_cast<int64_t>(k) * H) {
    const int64_t r = e / H;
    const int j = static_cast<int>(e % H);
    const double* xr = w.x + r * n_in;
    double acc = 0.0;
#pragma unroll 8
    for (int i = 0; i < n_in; ++i) acc = fma(xr[i], wv(a, static_cast<int64_t>(i) * H + j), acc);
    w.h[e] = tanh(__dadd_rn(acc, wv(a, static_cast<int64_t>(n_in) * H + j)));
  }
}

// 3. z = h @ W2 + b2: one CTA per (row, worker); the row of h and the W2 rows
// are staged through shared memory in chunks, so each class's long
// sequential chain (H fused multiply-adds) reads on-chip operands
__global__ void __launch_bounds__(kToyThreads) toy_logits_kernel(const __grid_constant__ ToyArgs a,
                                                                 int jc) {
  extern __shared__ __align__(16) double st[];
  const Work w = work_of(a, blockIdx.y);
  const int n_in = a.n_in, H = a.hidden, C = a.ncls;
  const int64_t r = blockIdx.x;
  const int64_t o_w2 = static_cast<int64_t>(n_in) * H + H;
  const int64_t o_b2 = o_w2 + static_cast<int64_t>(H) * C;
  double* hs = st;                                   // [jc]
  float* ws = reinterpret_cast<float*>(st + jc);     // [jc][C]
  const int tid = threadIdx.x, nt = blockDim.x;
  // each thread owns classes c = tid, tid + nt, ... (C is small: one pass)
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int c0 = 0; c0 < C; c0 += 4 * nt) {
    for (int j0 = 0; j0 < H; j0 += jc) {
      const int n = min(jc, H - j0);
      __syncthreads();
      for (int t = tid; t < n; t += nt) hs[t] = w.h[r * H + j0 + t];
      for (int t = tid; t < n * C; t += nt) ws[t] = __ldg(a.w + o_w2 + static_cast<int64_t>(j0) * C + t);
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = c0 + tid + q * nt;
        if (c < C) {
          double v = acc[q];
          // 16 operand pairs loaded ahead of their 16 chained multiply-adds
          int t = 0;
          for (; t + 16 <= n; t += 16) {
            double hv[16], wq[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              hv[u] = hs[t + u];
              wq[u] = static_cast<double>(ws[(t + u) * C + c]);
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) v = fma(hv[u], wq[u], v);
          }
          for (; t < n; ++t) v = fma(hs[t], static_cast<double>(ws[t * C + c]), v);
          acc[q] = v;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = c0 + tid + q * nt;
      if (c < C) w.pr[r * C + c] = __dadd_rn(acc[q], wv(a, o_b2 + c));
      acc[q] = 0.0;
    }
  }
}

// 4. per row: softmax, -log p[y], argmax, dz = p - onehot(y)
__global__ void __launch_bounds__(kToyThreads) toy_softmax_kernel(const __grid_constant__ ToyArgs a) {
  const Work w = work_of(a, blockIdx.y);
  const int k = a.batch, C = a.ncls;
  TOY_LOOP(r, k) {
    double* z = w.pr + r * C;
    double zmax = -INFINITY;
    for (int c = 0; c < C; ++c) zmax = fmax(zmax, z[c]);
    int arg = 0;
    for (int c = 0; c < C; ++c) {
      z[c] = __dsub_rn(z[c], zmax);
      if (z[c] > z[arg]) arg = c;
    }
    double s = -0.0;
    for (int c = 0; c < C; ++c) {
      z[c] = exp(z[c]);
      s = __dadd_rn(s, z[c]);
    }
    for (int c = 0; c < C; ++c) z[c] = __ddiv_rn(z[c], s);
    const int y = w.lab[r];
    w.lt[r] = -log(z[y]);
    if (arg == y) atomicAdd(w.correct, 1);
    z[y] = __dsub_rn(z[y], 1.0);
  }
}

// 5. da = (1 - h*h) * (dz @ W2.T)
__global__ void __launch_bounds__(kToyThreads) toy_dhidden_kernel(const __grid_constant__ ToyArgs a) {
  const Work w = work_of(a, blockIdx.y);
  const int k = a.batch, n_in = a.n_in, H = a.hidden, C = a.ncls;
  const int64_t o_w2 = static_cast<int64_t>(n_in) * H + H;
  TOY_LOOP(e, static_cast<int64_t>(k) * H) {
    const int64_t r = e / H;
    const int j = static_cast<int>(e % H);
    double acc = 0.0;
    for (int c = 0; c < C; ++c)
      acc = fma(w.pr[r * C + c], wv(a, o_w2 + static_cast<int64_t>(j) * C + c), acc);
    const double hv = w.h[e];
    w.da[e] = __dmul_rn(__dsub_rn(1.0, __dmul_rn(hv, hv)), acc);
  }
}

// 6. dW1 = x.T @ da, db1 = da.sum(0), dW2 = h.T @ dz, db2 = dz.sum(0); loss, count
__global__ void __launch_bounds__(kToyThreads) toy_params_kernel(const __grid_constant__ ToyArgs a) {
  const int wk = blockIdx.y;
  const Work w = work_of(a, wk);
  const int k = a.batch, n_in = a.n_in, H = a.hidden, C = a.ncls;
  const int64_t o_b1 = static_cast<int64_t>(n_in) * H, o_w2 = o_b1 + H;
  const int64_t o_b2 = o_w2 + static_cast<int64_t>(H) * C, p = o_b2 + C;
  float* out = a.out[wk];
  TOY_LOOP(e, p + 1) {
    if (e == p) {  // the tail slots: loss sum (numpy pairwise), correct count
      out[p] = __double2float_rn(__dadd_rn(0.0, np_pairwise(w.lt, k)));
      out[p + 1] = static_cast<float>(*w.correct);
      continue;
    }
    double acc = 0.0;
    if (e < o_b1) {
      const int64_t i = e / H, j = e % H;
#pragma unroll 8
      for (int r = 0; r < k; ++r) acc = fma(w.x[r * n_in + i], w.da[r * H + j], acc);
    } else if (e < o_w2) {
      const int64_t j = e - o_b1;
      for (int r = 0; r < k; ++r) acc = __dadd_rn(acc, w.da[r * H + j]);
    } else if (e < o_b2) {
      const int64_t j = (e - o_w2) / C, c = (e - o_w2) % C;
      for (int r = 0; r < k; ++r) acc = fma(w.h[r * H + j], w.pr[r * C + c], acc);
    } else {
      const int64_t c = e - o_b2;
      for (int r = 0; r < k; ++r) acc = __dadd_rn(acc, w.pr[r * C + c]);
    }
    out[e] = __double2float_rn(acc);
  }
}

unsigned blocks_for(int64_t elems) {
  const int64_t b = (elems + kToyThreads - 1) / kToyThreads;
  return static_cast<unsigned>(b < 1 ? 1 : (b > 4096 ? 4096 : b));
}

}  // namespace

}  // namespace md

extern "C" int64_t md_toy_work_bytes(int32_t n_in, int32_t hidden, int32_t n_classes,
                                     int32_t batch) {
  if (n_in < 1 || hidden < 1 || n_classes < 1 || batch < 1) return 0;
  return 8 * md::work_doubles(batch, n_in, hidden, n_classes) *
         static_cast<int64_t>(MD_MAX_WORKERS);
}

extern "C" int md_toy_grad(const float* w, int32_t n_in, int32_t hidden, int32_t n_classes,
                           const uint8_t* const* records, int32_t feature_bytes,
                           const int32_t* const* labels, int64_t record_stride, int32_t batch,
                           float* const* out, int32_t n_workers, double* work,
                           int64_t work_bytes, int32_t* status, void* stream) {
  if (!w || !records || !labels || !out || !work || n_in < 1 || hidden < 1 || n_classes < 1 ||
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
  const int64_t need = md_toy_work_bytes(n_in, hidden, n_classes, batch);
  if (work_bytes < need || (reinterpret_cast<uintptr_t>(work) & 7)) {
    md::set_error("md_toy_grad: workspace of %lld bytes (need %lld, 8-byte aligned)",
                  static_cast<long long>(work_bytes), static_cast<long long>(need));
    return MD_ERR_INVALID_CONFIG;
  }
  const int64_t k = batch, H = hidden, C = n_classes;
  const int64_t p = static_cast<int64_t>(n_in) * H + H + H * C + C;
  if (k > 65535) {
    md::set_error("md_toy_grad: batch %d exceeds 65535 rows", batch);
    return MD_ERR_INVALID_CONFIG;
  }
  // logits staging chunk: jc rows of h (float64) + W2 (float32) within 40 KB
  const int jc = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>(H, 40960 / (8 + 4 * C))));
  const size_t smem = static_cast<size_t>(jc) * 8 + static_cast<size_t>(jc) * C * 4;
  if (smem > 48 * 1024) {
    md::set_error("md_toy_grad: %d classes do not fit the logits staging", n_classes);
    return MD_ERR_INVALID_CONFIG;
  }
  cudaStream_t s = md::as_stream(stream);
  // worker chunks run one after another on the stream, so they share the workspace
  for (int32_t w0 = 0; w0 < n_workers; w0 += MD_MAX_WORKERS) {
    md::ToyArgs a{};
    a.w = w;
    a.n_in = n_in;
    a.hidden = hidden;
    a.ncls = n_classes;
    a.batch = batch;
    a.feature_bytes = feature_bytes;
    a.record_stride = record_stride;
    a.work_stride = md::work_doubles(k, n_in, H, C);
    a.work = work;
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
    const unsigned wm = static_cast<unsigned>(m);
    md::toy_input_kernel<<<dim3(md::blocks_for(std::max<int64_t>(k * n_in, k)), wm),
                           md::kToyThreads, 0, s>>>(a);
    MD_LAUNCH_CHECK();
    md::toy_hidden_kernel<<<dim3(md::blocks_for(k * H), wm), md::kToyThreads, 0, s>>>(a);
    MD_LAUNCH_CHECK();
    md::toy_logits_kernel<<<dim3(static_cast<unsigned>(k), wm), md::kToyThreads, smem, s>>>(a, jc);
    MD_LAUNCH_CHECK();
    md::toy_softmax_kernel<<<dim3(md::blocks_for(k), wm), md::kToyThreads, 0, s>>>(a);
    MD_LAUNCH_CHECK();
    md::toy_dhidden_kernel<<<dim3(md::blocks_for(k * H), wm), md::kToyThreads, 0, s>>>(a);
    MD_LAUNCH_CHECK();
    md::toy_params_kernel<<<dim3(md::blocks_for(p + 1), wm), md::kToyThreads, 0, s>>>(a);
    MD_LAUNCH_CHECK();
  }
  return MD_OK;
}
