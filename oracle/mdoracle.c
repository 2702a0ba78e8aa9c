/*
 * mdoracle.c -- CPU restatement of the reference's data-parallel hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline -- never as the product path.
 *
 * Every function restates /root/reference/pkg/src/minidist/ (cited per
 * function) in plain C, built with -ffp-contract=off like the reference's
 * kernels (pkg/setup.py:31-32) so float results are bit-comparable.
 * The RNG restates numpy 2.x's Philox4x64-10 / Generator.integers /
 * Generator.permutation (numpy is the reference's unvendored dependency,
 * pkg/pyproject.toml:11; the restatement is checked against numpy itself in
 * tests/test_oracle.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- float kernels: _kernels/_accel.pyx:12-29, fallback.py:6-23 ---------- */
void mo_add_f32(float* dst, const float* src, int64_t n) {
  for (int64_t i = 0; i < n; ++i) dst[i] = dst[i] + src[i];
}

void mo_sub_scaled_f32(float* dst, const float* src, int64_t n, double c) {
  const float cf = (float)c; /* Cython `float c` parameter */
  for (int64_t i = 0; i < n; ++i) {
    float p = cf * src[i];
    dst[i] = dst[i] - p;
  }
}

/* Momentum / weight-decay extension (NOT in the reference; see mdb200.h). */
void mo_sgd_update(float* w, const float* g, float* mom, int64_t n, float c, float mu,
                   float wd_b) {
  for (int64_t i = 0; i < n; ++i) {
    float d = g[i];
    if (wd_b != 0.0f) {
      float t = wd_b * w[i];
      d = d + t;
    }
    if (mom) {
      float t = mu * mom[i];
      float v = t + d;
      mom[i] = v;
      d = v;
    }
    float p = c * d;
    w[i] = w[i] - p;
  }
}

/* bench.py:188-195 (_fill_rank_input) */
void mo_fill_rank_input(float* buf, int64_t n, int rank, int n_ranks) {
  double scale = ((double)rank + 1.0) * 3.141592653589793 / (double)n_ranks;
  for (int64_t i = 0; i < n; ++i) buf[i] = (float)(((double)(i % 997) + 1.0) * scale);
}

/* ---- fold trees: collectives.py:271-296, pkg/tests/oracles.py:17-76 --------
 * CSR tables as in md_plan_create (include/mdb200.h). fold(node) = own value
 * at position self_pos among the node's children's subtree folds, added left
 * to right. out[lo:hi] = fold(root of color c) over chunk c. */
static void fold_node(int n, const int32_t* cptr, const int32_t* cidx, const int32_t* spos,
                      int row0, int node, const float* const* in, int64_t lo, int64_t hi,
                      float* acc, float* tmp_pool, int depth) {
  int row = row0 + node;
  int nk = cptr[row + 1] - cptr[row];
  int sp = spos ? spos[row] : 0;
  int64_t len = hi - lo;
  float* tmp = tmp_pool + (int64_t)depth * len;
  int first = 1;
  for (int j = 0, q = 0; j <= nk; ++j) {
    const float* src;
    if (j == sp) {
      src = in[node] + lo;
    } else {
      fold_node(n, cptr, cidx, spos, row0, cidx[cptr[row] + q], in, lo, hi, tmp, tmp_pool,
                depth + 1);
      ++q;
      src = tmp;
    }
    if (first) {
      memcpy(acc, src, (size_t)len * sizeof(float));
      first = 0;
    } else {
      for (int64_t i = 0; i < len; ++i) acc[i] = acc[i] + src[i];
    }
  }
}

static int root_of(int n, const int32_t* parent, int row0) {
  for (int r = 0; r < n; ++r)
    if (parent[row0 + r] < 0) return r;
  return -1;
}

/* Fold [lo, hi) of the payload: result into out (length hi - lo).
 * tmp_pool: (n + 1) * (hi - lo) floats of scratch. */
void mo_fold_range(int n, int k, const int32_t* parent, const int32_t* cptr, const int32_t* cidx,
                   const int32_t* spos, const float* const* in, int64_t total, int64_t lo,
                   int64_t hi, float* out, float* tmp_pool) {
  int64_t base = total / k, extra = total % k;
  for (int c = 0; c < k; ++c) {
    int64_t cs = c * base + (c < extra ? c : extra);
    int64_t ce = cs + base + (c < extra ? 1 : 0);
    int64_t a = cs > lo ? cs : lo, b = ce < hi ? ce : hi;
    if (a >= b) continue;
    int row0 = c * n;
    fold_node(n, cptr, cidx, spos, row0, root_of(n, parent, row0), in, a, b, out + (a - lo),
              tmp_pool, 0);
  }
}

/* ---- threaded allreduce port (the CPU baseline of bench.py) ----------------
 * Ranks' buffers bufs[0..n) are summed per element in the tree fold order and
 * the result broadcast into every buffer (collectives.py:225-296); optional
 * fused SGD update of per-rank weights. Work is split across `threads` host
 * threads by element range. */
typedef struct {
  int n, k;
  const int32_t *parent, *cptr, *cidx, *spos;
  float* const* bufs;
  int64_t total, lo, hi;
  float* const* w;
  float* const* mom;
  int64_t update_len;
  float c, mu, wd_b;
} fold_job;

static void* fold_worker(void* arg) {
  fold_job* j = (fold_job*)arg;
  const int64_t chunk = 16384;
  float* out = (float*)malloc(sizeof(float) * chunk);
  float* pool = (float*)malloc(sizeof(float) * chunk * (j->n + 1));
  for (int64_t lo = j->lo; lo < j->hi; lo += chunk) {
    int64_t hi = lo + chunk < j->hi ? lo + chunk : j->hi;
    mo_fold_range(j->n, j->k, j->parent, j->cptr, j->cidx, j->spos, (const float* const*)j->bufs,
                  j->total, lo, hi, out, pool);
    for (int r = 0; r < j->n; ++r) {
      memcpy(j->bufs[r] + lo, out, sizeof(float) * (size_t)(hi - lo));
      if (j->w && lo < j->update_len) {
        int64_t uh = hi < j->update_len ? hi : j->update_len;
        mo_sgd_update(j->w[r] + lo, out, j->mom ? j->mom[r] + lo : NULL, uh - lo, j->c, j->mu,
                      j->wd_b);
      }
    }
  }
  free(out);
  free(pool);
  return NULL;
}

int mo_allreduce_threads(int n, int k, const int32_t* parent, const int32_t* cptr,
                         const int32_t* cidx, const int32_t* spos, float* const* bufs,
                         int64_t total, float* const* w, float* const* mom, int64_t update_len,
                         float c, float mu, float wd_b, int threads) {
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  fold_job* jobs = (fold_job*)malloc(sizeof(fold_job) * threads);
  int64_t per = (total + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    fold_job* j = &jobs[t];
    j->n = n;
    j->k = k;
    j->parent = parent;
    j->cptr = cptr;
    j->cidx = cidx;
    j->spos = spos;
    j->bufs = bufs;
    j->total = total;
    j->lo = (int64_t)t * per < total ? (int64_t)t * per : total;
    j->hi = (int64_t)(t + 1) * per < total ? (int64_t)(t + 1) * per : total;
    j->w = w;
    j->mom = mom;
    j->update_len = update_len;
    j->c = c;
    j->mu = mu;
    j->wd_b = wd_b;
    pthread_create(&th[t], NULL, fold_worker, j);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}

/* ---- numpy Philox4x64-10 / Generator semantics ------------------------------ */
static inline void mulhilo(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
  unsigned __int128 p = (unsigned __int128)a * b;
  *lo = (uint64_t)p;
  *hi = (uint64_t)(p >> 64);
}

void mo_philox_block(uint64_t ctr0, uint64_t key, uint64_t out[4]) {
  uint64_t v0 = ctr0, v1 = 0, v2 = 0, v3 = 0, k0 = key, k1 = 0;
  for (int r = 0; r < 10; ++r) {
    uint64_t h0, l0, h1, l1;
    mulhilo(0xD2E7470EE14C6C93ULL, v0, &h0, &l0);
    mulhilo(0xCA5A826395121157ULL, v2, &h1, &l1);
    uint64_t a = h1 ^ v1 ^ k0, b = h0 ^ v3 ^ k1;
    v0 = a;
    v1 = l1;
    v2 = b;
    v3 = l0;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  out[0] = v0;
  out[1] = v1;
  out[2] = v2;
  out[3] = v3;
}

/* Sequential stream of a fresh Generator(Philox(key)): 64-bit words consumed
 * in order (counter pre-incremented), 32-bit draws low half then high half. */
typedef struct {
  uint64_t key, ctr;
  uint64_t blk[4];
  int pos;   /* next u64 in blk (4 = empty) */
  int has32; /* buffered high half */
  uint32_t buf32;
} mo_rng;

static void rng_init(mo_rng* g, uint64_t key) {
  g->key = key;
  g->ctr = 0;
  g->pos = 4;
  g->has32 = 0;
}
static uint64_t rng_next64(mo_rng* g) {
  if (g->pos == 4) {
    g->ctr += 1;
    mo_philox_block(g->ctr, g->key, g->blk);
    g->pos = 0;
  }
  return g->blk[g->pos++];
}
static uint32_t rng_next32(mo_rng* g) {
  if (g->has32) {
    g->has32 = 0;
    return g->buf32;
  }
  uint64_t w = rng_next64(g);
  g->has32 = 1;
  g->buf32 = (uint32_t)(w >> 32);
  return (uint32_t)w;
}

/* Generator.integers(0, n, size) for 1 <= n <= 2^32 (Lemire, 32-bit). */
void mo_integers(uint64_t key, uint64_t n, int64_t size, int64_t* out) {
  mo_rng g;
  rng_init(&g, key);
  if (n == 1) {
    memset(out, 0, sizeof(int64_t) * (size_t)size);
    return;
  }
  uint32_t rng_excl = (uint32_t)n;
  for (int64_t i = 0; i < size; ++i) {
    if (n == 0x100000000ULL) {
      out[i] = rng_next32(&g);
      continue;
    }
    uint64_t m = (uint64_t)rng_next32(&g) * rng_excl;
    uint32_t left = (uint32_t)m;
    if (left < rng_excl) {
      uint32_t thr = (uint32_t)((0x100000000ULL - rng_excl) % rng_excl);
      while (left < thr) {
        m = (uint64_t)rng_next32(&g) * rng_excl;
        left = (uint32_t)m;
      }
    }
    out[i] = (int64_t)(m >> 32);
  }
}

/* Generator.permutation(n): Fisher-Yates, i = n-1 .. 1, j = random_interval(i). */
void mo_permutation(uint64_t key, int64_t n, int64_t* out) {
  mo_rng g;
  rng_init(&g, key);
  for (int64_t i = 0; i < n; ++i) out[i] = i;
  for (int64_t i = n - 1; i >= 1; --i) {
    uint64_t mask = (uint64_t)i;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    mask |= mask >> 32;
    uint64_t v;
    if ((uint64_t)i <= 0xFFFFFFFFULL) {
      while ((v = (rng_next32(&g) & mask)) > (uint64_t)i) {
      }
    } else {
      while ((v = (rng_next64(&g) & mask)) > (uint64_t)i) {
      }
    }
    int64_t t = out[i];
    out[i] = out[v];
    out[v] = t;
  }
}

/* dimd.py:226-234 */
uint64_t mo_mix64(const uint64_t* parts, int n) {
  uint64_t acc = 0;
  for (int i = 0; i < n; ++i) {
    acc = acc + parts[i] + 0x9E3779B97F4A7C15ULL;
    acc = (acc ^ (acc >> 30)) * 0xBF58476D1CE4E5B9ULL;
    acc = (acc ^ (acc >> 27)) * 0x94D049BB133111EBULL;
    acc ^= acc >> 31;
  }
  return acc;
}

/* ---- shuffle index plan: dimd.py:281-339, for one receiving member ----------
 * n_rec[S]: record counts of the group members. Writes (member, record) of
 * every output slot in final order; returns N'. out arrays need sum(n_rec). */
int64_t mo_shuffle_plan(uint64_t seed, uint64_t group_id, int S, int member, uint64_t global_rank,
                        int64_t m, const int64_t* n_rec, int32_t* out_member, int64_t* out_rec) {
  const uint64_t DEST = 0x74736564ULL, PERM = 0x6d726570ULL;
  int64_t total = 0;
  for (int q = 0; q < S; ++q) total += n_rec[q];
  int32_t* got_m = (int32_t*)malloc(sizeof(int32_t) * (size_t)(total + 1));
  int64_t* got_r = (int64_t*)malloc(sizeof(int64_t) * (size_t)(total + 1));
  int64_t nf = 0;
  int64_t maxn = 1;
  for (int q = 0; q < S; ++q)
    if (n_rec[q] > maxn) maxn = n_rec[q];
  int64_t* dests = (int64_t*)malloc(sizeof(int64_t) * (size_t)maxn);
  for (int64_t t = 0; t < m; ++t) {
    for (int q = 0; q < S; ++q) { /* alltoallv receive order: source rank ascending */
      int64_t n = n_rec[q];
      int64_t lo = t * n / m, hi = (t + 1) * n / m;
      if (hi <= lo) continue;
      uint64_t parts[5] = {seed, DEST, group_id, (uint64_t)q, (uint64_t)t};
      mo_integers(mo_mix64(parts, 5), (uint64_t)S, hi - lo, dests);
      for (int64_t i = lo; i < hi; ++i) /* flatnonzero: stable, source order */
        if (dests[i - lo] == member) {
          got_m[nf] = q;
          got_r[nf] = i;
          ++nf;
        }
    }
  }
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nf + 1));
  uint64_t pp[3] = {seed, PERM, global_rank};
  mo_permutation(mo_mix64(pp, 3), nf, perm);
  for (int64_t i = 0; i < nf; ++i) {
    out_member[i] = got_m[perm[i]];
    out_rec[i] = got_r[perm[i]];
  }
  free(perm);
  free(dests);
  free(got_m);
  free(got_r);
  return nf;
}

/* random_batch picks, dimd.py:213-220 */
void mo_random_batch(uint64_t key, int64_t n_records, int64_t batch, int64_t* picks) {
  mo_integers(key, (uint64_t)n_records, batch, picks);
}

/* ---- the reference's gradient producer: ToyModel.loss_and_grad_sum ---------
 * sgd.py:148-248: one-hidden-layer tanh MLP + softmax cross entropy, all math
 * in float64 from the float32 weights, gradient rounded to float32 once.
 * numpy's float64 matmul (OpenBLAS dgemm) accumulates every output element
 * over the inner index in order with fused multiply-adds (measured against
 * numpy here for batch >= 2); row sums of exp are sequential (numpy's pairwise
 * sum is sequential below 8 terms), column sums (axis 0) sequential over
 * rows, the loss sum numpy's pairwise sum. Weights [W1 | b1 | W2 | b2]. */
static double np_pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double r = -0.0;
    for (int64_t i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    int64_t i;
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
}

/* x: [k][n_in] float32 record values; y: labels; out: p + 2 floats
 * (gradient sum, loss sum, correct count -- node_gradient's buffer, sgd.py:335-353) */
void mo_toy_grad(const float* w, int n_in, int hidden, int ncls, const float* x,
                 const int64_t* y, int k, float* out) {
  const int o_b1 = n_in * hidden, o_w2 = o_b1 + hidden, o_b2 = o_w2 + hidden * ncls;
  const int p = o_b2 + ncls;
  double* h = (double*)malloc(sizeof(double) * (size_t)k * hidden);
  double* pr = (double*)malloc(sizeof(double) * (size_t)k * ncls);
  double* zz = (double*)malloc(sizeof(double) * (size_t)k * ncls);
  double* da = (double*)malloc(sizeof(double) * (size_t)k * hidden);
  double* lt = (double*)malloc(sizeof(double) * (size_t)(k + 1));
  int64_t correct = 0;
  for (int r = 0; r < k; ++r) {
    for (int j = 0; j < hidden; ++j) { /* h = tanh(x @ W1 + b1) */
      double acc = 0.0;
      for (int i = 0; i < n_in; ++i) acc = fma((double)x[r * n_in + i], (double)w[i * hidden + j], acc);
      h[r * hidden + j] = tanh(acc + (double)w[o_b1 + j]);
    }
    double zmax = -INFINITY;
    for (int c = 0; c < ncls; ++c) { /* z = h @ W2 + b2 */
      double acc = 0.0;
      for (int j = 0; j < hidden; ++j) acc = fma(h[r * hidden + j], (double)w[o_w2 + j * ncls + c], acc);
      zz[r * ncls + c] = acc + (double)w[o_b2 + c];
      if (zz[r * ncls + c] > zmax) zmax = zz[r * ncls + c];
    }
    double s = -0.0;
    int arg = 0;
    for (int c = 0; c < ncls; ++c) {
      zz[r * ncls + c] = zz[r * ncls + c] - zmax;
      if (zz[r * ncls + c] > zz[r * ncls + arg]) arg = c; /* argmax: first maximum */
      pr[r * ncls + c] = exp(zz[r * ncls + c]);
      s += pr[r * ncls + c];
    }
    for (int c = 0; c < ncls; ++c) pr[r * ncls + c] = pr[r * ncls + c] / s;
    lt[r] = -log(pr[r * ncls + y[r]]);
    correct += (arg == y[r]);
    pr[r * ncls + y[r]] -= 1.0; /* dz */
  }
  double loss = 0.0 + np_pairwise(lt, k);
  for (int r = 0; r < k; ++r) /* dh = dz @ W2.T; da = (1 - h*h) * dh */
    for (int j = 0; j < hidden; ++j) {
      double acc = 0.0;
      for (int c = 0; c < ncls; ++c) acc = fma(pr[r * ncls + c], (double)w[o_w2 + j * ncls + c], acc);
      double hv = h[r * hidden + j];
      da[r * hidden + j] = (1.0 - hv * hv) * acc;
    }
  for (int i = 0; i < n_in; ++i) /* dW1 = x.T @ da */
    for (int j = 0; j < hidden; ++j) {
      double acc = 0.0;
      for (int r = 0; r < k; ++r) acc = fma((double)x[r * n_in + i], da[r * hidden + j], acc);
      out[i * hidden + j] = (float)acc;
    }
  for (int j = 0; j < hidden; ++j) { /* db1 = da.sum(0) */
    double acc = 0.0;
    for (int r = 0; r < k; ++r) acc += da[r * hidden + j];
    out[o_b1 + j] = (float)acc;
  }
  for (int j = 0; j < hidden; ++j) /* dW2 = h.T @ dz */
    for (int c = 0; c < ncls; ++c) {
      double acc = 0.0;
      for (int r = 0; r < k; ++r) acc = fma(h[r * hidden + j], pr[r * ncls + c], acc);
      out[o_w2 + j * ncls + c] = (float)acc;
    }
  for (int c = 0; c < ncls; ++c) { /* db2 = dz.sum(0) */
    double acc = 0.0;
    for (int r = 0; r < k; ++r) acc += pr[r * ncls + c];
    out[o_b2 + c] = (float)acc;
  }
  out[p] = (float)loss;
  out[p + 1] = (float)correct;
  free(h);
  free(pr);
  free(zz);
  free(da);
  free(lt);
}
