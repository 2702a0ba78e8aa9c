// Multi-color tree allreduce over NVLink/NVSwitch peer memory (sm_100a).
//
// Reference semantics (/root/reference/pkg/src/minidist/collectives.py):
//   * allreduce_multicolor (:225-268): the payload is split into k contiguous
//     chunks (make_chunk_plan, topology.py:103-120); chunk c is reduced up
//     color tree c -- every node folds, IN CHILD-LIST ORDER, its own value and
//     its children's subtree sums (_tree_up_task, :271-286) -- and the root's
//     result is broadcast back down the same tree (_tree_down_task, :289-296).
//   * allreduce_ring (:302-359) is the same fold on a chain (each node folds
//     its successor), reduce_then_broadcast (:365-409) a star whose root folds
//     every rank in ascending rank order. All three are one kernel here; the
//     fold tree is data (md_plan_t).
//
// B200 design: ONE persistent kernel per call and rank, picked per call
// (md_allreduce_ex; md_plan_set_route pins one): LL push, one-shot pull,
// owner-push (plain calls and the sharded SGD update), the tiled all-pull
// stream kernel, the channelized tree and the work-queue tree. The tree
// kernels move each color's chunk along its tree (UP folds in the reference
// order with __fadd_rn, DOWN copies the parent's final); the others evaluate
// each color's fold program (the same adds in the same order) on data pulled
// or pushed over NVLink. The optional prologue folds per-worker gradient
// buffers (sgd.py:335-353) into the own value, and the optional epilogue
// applies the SGD (momentum / weight-decay) update as soon as a segment's
// sum is final, so the gradient is never re-read from HBM.
//
// Synchronisation (replaces the transport's expose/pull and the length-header
// barrier of _check_same_length, :157-174): epoch-tagged flags in peer-mapped
// control blocks, polled with ld.acquire.sys (published as described at
// publish_flags); an entry barrier carries every rank's
// buffer length (LengthMismatch) and route word (InvalidConfig) and an exit
// barrier guarantees no peer still reads a buffer when the call returns.
// Waits are bounded by a globaltimer watchdog (NotExposed). No flag is ever
// reset: epochs only grow.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include "md_allreduce.cuh"

namespace md {

struct TraceBuf {
  void* ptr = nullptr;
  size_t bytes = 0, used = 0;
};
static TraceBuf g_trace[64];

// ---- plan construction (host) ------------------------------------------------
static int build_rank_plans(int n, int k, const int32_t* parent, const int32_t* child_ptr,
                            const int32_t* child_idx, const int32_t* self_pos,
                            std::vector<RankPlan>* out) {
  out->assign(n, RankPlan{});
  for (int c = 0; c < k; ++c) {
    const int32_t* par = parent + c * n;
    int root = -1;
    for (int r = 0; r < n; ++r) {
      if (par[r] < -1 || par[r] >= n || par[r] == r) {
        set_error("color %d: bad parent %d of rank %d", c, par[r], r);
        return MD_ERR_INVALID_CONFIG;
      }
      if (par[r] == -1) {
        if (root >= 0) {
          set_error("color %d has two roots (%d, %d)", c, root, r);
          return MD_ERR_INVALID_CONFIG;
        }
        root = r;
      }
    }
    if (root < 0) {
      set_error("color %d has no root", c);
      return MD_ERR_INVALID_CONFIG;
    }
    auto kids = [&](int r, int* cnt) {
      int row = c * n + r;
      *cnt = child_ptr[row + 1] - child_ptr[row];
      return child_idx + child_ptr[row];
    };
    // consistency + acyclicity: depth via parent chain (<= n steps)
    std::vector<int> depth(n, -1), height(n, 0);
    for (int r = 0; r < n; ++r) {
      int d = 0, cur = r;
      while (par[cur] >= 0 && d <= n) {
        cur = par[cur];
        ++d;
      }
      if (d > n || cur != root) {
        set_error("color %d: cycle reachable from rank %d", c, r);
        return MD_ERR_INVALID_CONFIG;
      }
      depth[r] = d;
      int cnt;
      const int32_t* ch = kids(r, &cnt);
      if (cnt < 0 || cnt > MD_MAX_RANKS) {
        set_error("color %d: rank %d has %d children", c, r, cnt);
        return MD_ERR_INVALID_CONFIG;
      }
      for (int j = 0; j < cnt; ++j) {
        if (ch[j] < 0 || ch[j] >= n || par[ch[j]] != r) {
          set_error("color %d: child %d of %d disagrees with parent map", c, ch[j], r);
          return MD_ERR_INVALID_CONFIG;
        }
      }
    }
    int total_children = 0;
    for (int r = 0; r < n; ++r) {
      int cnt;
      kids(r, &cnt);
      total_children += cnt;
    }
    if (total_children != n - 1) {
      set_error("color %d: children lists cover %d ranks, expected %d", c, total_children, n - 1);
      return MD_ERR_INVALID_CONFIG;
    }
    // heights, deepest first
    std::vector<int> order(n);
    for (int r = 0; r < n; ++r) order[r] = r;
    std::sort(order.begin(), order.end(), [&](int x, int y) { return depth[x] > depth[y]; });
    for (int r : order)
      if (par[r] >= 0) height[par[r]] = std::max(height[par[r]], height[r] + 1);
    const int H = height[root];

    auto fold_pos = [&](int r) { return self_pos ? self_pos[c * n + r] : 0; };
    for (int r = 0; r < n; ++r) {
      RankPlan& rp = (*out)[r];
      int cnt;
      const int32_t* ch = kids(r, &cnt);
      int sp = fold_pos(r);
      if (sp < 0 || sp > cnt) {
        set_error("color %d: self position %d out of range for rank %d", c, sp, r);
        return MD_ERR_INVALID_CONFIG;
      }
      Task up{};
      up.type = 0;
      up.color = c;
      up.stage = height[r];
      up.parent = par[r];
      up.is_leaf = cnt == 0;
      up.n_fold = cnt + 1;
      for (int j = 0, q = 0; j <= cnt; ++j) {
        if (j == sp) {
          up.fold_src[j] = r;
          up.fold_leaf[j] = 0;
        } else {
          int chr = ch[q++];
          up.fold_src[j] = chr;
          int gc;
          kids(chr, &gc);
          up.fold_leaf[j] = gc == 0;
        }
      }
      if (par[r] >= 0) {
        int pcnt;
        const int32_t* pch = kids(par[r], &pcnt);
        int ci = 0;
        while (ci < pcnt && pch[ci] != r) ++ci;
        int psp = fold_pos(par[r]);
        up.my_slot = ci >= psp ? ci + 1 : ci;
      } else {
        up.n_down = cnt;
        for (int j = 0; j < cnt; ++j) up.down[j] = ch[j];
      }
      rp.t[rp.n_tasks++] = up;
      if (par[r] >= 0) {
        Task dn{};
        dn.type = 1;
        dn.color = c;
        dn.stage = H + depth[r];
        dn.parent = par[r];
        dn.n_down = cnt;
        for (int j = 0; j < cnt; ++j) dn.down[j] = ch[j];
        rp.t[rp.n_tasks++] = dn;
      }
    }
  }
  for (auto& rp : *out)
    std::stable_sort(rp.t, rp.t + rp.n_tasks,
                     [](const Task& x, const Task& y) { return x.stage < y.stage; });
  return MD_OK;
}

// Each color's fold as a post-order program over rank slots (ColorProg), from
// the same per-rank UP tasks the tree schedule runs: op = (folding rank, its
// fold list), ordered by subtree height so children come before parents.
static void build_fold_prog(const std::vector<RankPlan>& plans, int n, int k, FoldProg* out) {
  memset(out, 0, sizeof(*out));
  for (int c = 0; c < k; ++c) {
    ColorProg& p = out->c[c];
    std::vector<std::pair<int, const Task*>> ops;  // (folding rank, its UP task)
    for (int r = 0; r < n; ++r)
      for (int i = 0; i < plans[r].n_tasks; ++i) {
        const Task& t = plans[r].t[i];
        if (t.type != 0 || t.color != c) continue;
        if (t.parent < 0) p.root = static_cast<uint8_t>(r);
        if (t.n_fold > 1) ops.push_back({r, &t});
      }
    std::stable_sort(ops.begin(), ops.end(), [](const auto& x, const auto& y) {
      return x.second->stage < y.second->stage;
    });
    int off = 0;
    for (const auto& [r, t] : ops) {
      p.op_dst[p.n_ops] = static_cast<uint8_t>(r);
      p.op_cnt[p.n_ops] = static_cast<uint8_t>(t->n_fold);
      for (int j = 0; j < t->n_fold; ++j) p.items[off++] = static_cast<uint8_t>(t->fold_src[j]);
      ++p.n_ops;
    }
  }
}

// Owner-computes schedule ("which data movement"): the
// buffer is cut into n equal slices (chunk_of with n "colors"); rank j owns
// slice j: it pulls every rank's slice j and evaluates each element's OWN
// color fold program (task type 2), then every other rank copies the final
// slice from j (DOWN). Same adds in the same order per element as the tree
// schedule -- same bits -- but every rank ingests 2 (n-1)/n of the buffer for
// any k, where the reference's trees cap k = 1 / 2 at N = 4 at 50 / 75 %.
static void build_owner_plans(int n, std::vector<RankPlan>* out) {
  out->assign(n, RankPlan{});
  for (int j = 0; j < n; ++j) {
    for (int r = 0; r < n; ++r) {
      RankPlan& rp = (*out)[r];
      Task t{};
      t.color = j;
      if (r == j) {
        t.type = 2;
        t.stage = 0;
        t.parent = -1;
        t.n_fold = n;
        for (int q = 0; q < n; ++q) {
          t.fold_src[q] = q;
          t.fold_leaf[q] = 1;  // raw inputs: ready at the entry barrier
        }
        t.n_down = n - 1;
        for (int q = 0, c = 0; q < n; ++q)
          if (q != j) t.down[c++] = q;
      } else {
        t.type = 1;
        t.stage = 1;
        t.parent = j;
        t.n_down = 0;
      }
      rp.t[rp.n_tasks++] = t;
    }
  }
  for (auto& rp : *out)
    std::stable_sort(rp.t, rp.t + rp.n_tasks,
                     [](const Task& x, const Task& y) { return x.stage < y.stage; });
}

}  // namespace md

using namespace md;

extern "C" {

int md_device_count(int* n) {
  MD_CUDA_TRY(cudaGetDeviceCount(n));
  return MD_OK;
}

int md_enable_peer_access(int dev, int peer) {
  if (dev == peer) return MD_OK;
  int prev;
  MD_CUDA_TRY(cudaGetDevice(&prev));
  MD_CUDA_TRY(cudaSetDevice(dev));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    e = cudaSuccess;
  }
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    set_error("cudaDeviceEnablePeerAccess(%d -> %d): %s", dev, peer, cudaGetErrorString(e));
    return MD_ERR_CUDA;
  }
  return MD_OK;
}

typedef int (*PFN_getAddressRange)(unsigned long long*, size_t*, unsigned long long);

int md_mem_export(const void* ptr, unsigned char handle[MD_IPC_HANDLE_BYTES], uint64_t* offset) {
  static PFN_getAddressRange fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    MD_CUDA_TRY(cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q));
    if (!p) {
      set_error("cuMemGetAddressRange unavailable");
      return MD_ERR_CUDA;
    }
    fn = reinterpret_cast<PFN_getAddressRange>(p);
  }
  unsigned long long base = 0;
  size_t size = 0;
  int rc = fn(&base, &size, reinterpret_cast<unsigned long long>(ptr));
  if (rc != 0) {
    set_error("cuMemGetAddressRange failed (%d)", rc);
    return MD_ERR_CUDA;
  }
  cudaIpcMemHandle_t h;
  MD_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  static_assert(sizeof(h) == MD_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle, &h, sizeof(h));
  *offset = reinterpret_cast<unsigned long long>(ptr) - base;
  return MD_OK;
}

int md_mem_import(const unsigned char handle[MD_IPC_HANDLE_BYTES], void** base) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  MD_CUDA_TRY(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
  return MD_OK;
}

int md_mem_close(void* base) {
  MD_CUDA_TRY(cudaIpcCloseMemHandle(base));
  return MD_OK;
}

int md_comm_create(int32_t rank, int32_t n_ranks, int32_t device, md_comm_t** out) {
  if (n_ranks < 1 || n_ranks > MD_MAX_RANKS || rank < 0 || rank >= n_ranks) {
    set_error("rank %d of %d unsupported (max %d ranks)", rank, n_ranks, MD_MAX_RANKS);
    return MD_ERR_INVALID_CONFIG;
  }
  int prev;
  MD_CUDA_TRY(cudaGetDevice(&prev));
  MD_CUDA_TRY(cudaSetDevice(device));
  md_comm* c = new md_comm();
  c->rank = rank;
  c->n_ranks = n_ranks;
  c->device = device;
  c->epoch = 0;
  c->timeout_s = 30.0;
  cudaError_t e = cudaMalloc(&c->ctrl, sizeof(Ctrl));
  if (e == cudaSuccess) e = cudaMemset(c->ctrl, 0, sizeof(Ctrl));
  if (e == cudaSuccess) e = cudaHostAlloc(&c->err_host, 2 * sizeof(int32_t), cudaHostAllocMapped);
  if (e == cudaSuccess) {
    c->err_host[0] = c->err_host[1] = 0;
    e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->err_dev), c->err_host, 0);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    set_error("md_comm_create: %s", cudaGetErrorString(e));
    delete c;
    return MD_ERR_CUDA;
  }
  for (int r = 0; r < MD_MAX_RANKS; ++r) c->peer_ctrl[r] = nullptr;
  c->peer_ctrl[rank] = c->ctrl;
  *out = c;
  return MD_OK;
}

int md_comm_destroy(md_comm_t* c) {
  if (!c) return MD_OK;
  int prev;
  cudaGetDevice(&prev);
  cudaSetDevice(c->device);
  cudaFree(c->ctrl);
  cudaFreeHost(c->err_host);
  cudaSetDevice(prev);
  delete c;
  return MD_OK;
}

int md_comm_ctrl_ptr(md_comm_t* c, void** ctrl) {
  *ctrl = c->ctrl;
  return MD_OK;
}

int md_comm_set_peer_ctrl(md_comm_t* c, void* const* ptrs, int32_t n) {
  if (n != c->n_ranks) {
    set_error("expected %d control pointers, got %d", c->n_ranks, n);
    return MD_ERR_INVALID_CONFIG;
  }
  for (int r = 0; r < n; ++r)
    c->peer_ctrl[r] = (r == c->rank) ? c->ctrl : static_cast<Ctrl*>(ptrs[r]);
  return MD_OK;
}

int md_comm_take_error(md_comm_t* c, int32_t* code, int32_t* detail) {
  volatile int32_t* e = c->err_host;
  *code = e[0];
  *detail = e[1];
  e[0] = 0;
  e[1] = 0;
  return MD_OK;
}

int md_comm_set_timeout(md_comm_t* c, double seconds) {
  if (!(seconds > 0)) {
    set_error("timeout must be > 0");
    return MD_ERR_INVALID_CONFIG;
  }
  c->timeout_s = seconds;
  return MD_OK;
}

int md_plan_create(int32_t n_ranks, int32_t k, const int32_t* parent, const int32_t* child_ptr,
                   const int32_t* child_idx, const int32_t* self_pos, int32_t device,
                   md_plan_t** out) {
  if (n_ranks < 1 || n_ranks > MD_MAX_RANKS) {
    set_error("n_ranks %d unsupported (max %d)", n_ranks, MD_MAX_RANKS);
    return MD_ERR_INVALID_CONFIG;
  }
  if (k < 1 || k > MD_MAX_COLORS) {
    set_error("%d colors unsupported (max %d)", k, MD_MAX_COLORS);
    return MD_ERR_INVALID_CONFIG;
  }
  std::vector<RankPlan> host;
  int rc = build_rank_plans(n_ranks, k, parent, child_ptr, child_idx, self_pos, &host);
  if (rc != MD_OK) return rc;
  int prev;
  MD_CUDA_TRY(cudaGetDevice(&prev));
  MD_CUDA_TRY(cudaSetDevice(device));
  md_plan* p = new md_plan();
  p->n_ranks = n_ranks;
  p->k = k;
  p->device = device;
  p->host = host;
  p->prog_dev = nullptr;
  p->owner_dev = nullptr;
  p->schedule = MD_SCHED_TREE;
  p->route = MD_ROUTE_AUTO;
  p->tile = 0;
  FoldProg prog;
  build_fold_prog(host, n_ranks, k, &prog);
  build_owner_plans(n_ranks, &p->owner_host);
  cudaError_t e = cudaMalloc(&p->dev, sizeof(RankPlan) * n_ranks);
  if (e == cudaSuccess)
    e = cudaMemcpy(p->dev, host.data(), sizeof(RankPlan) * n_ranks, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&p->prog_dev, sizeof(FoldProg));
  if (e == cudaSuccess) e = cudaMemcpy(p->prog_dev, &prog, sizeof(FoldProg), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&p->owner_dev, sizeof(RankPlan) * n_ranks);
  if (e == cudaSuccess)
    e = cudaMemcpy(p->owner_dev, p->owner_host.data(), sizeof(RankPlan) * n_ranks,
                   cudaMemcpyHostToDevice);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    set_error("md_plan_create: %s", cudaGetErrorString(e));
    delete p;
    return MD_ERR_CUDA;
  }
  *out = p;
  return MD_OK;
}

int md_plan_set_schedule(md_plan_t* p, int32_t schedule) {
  if (!p || (schedule != MD_SCHED_TREE && schedule != MD_SCHED_OWNER)) {
    set_error("bad plan or schedule %d", schedule);
    return MD_ERR_INVALID_CONFIG;
  }
  p->schedule = schedule;
  return MD_OK;
}

int md_plan_set_route(md_plan_t* p, int32_t route, int64_t tile) {
  if (!p || route < MD_ROUTE_AUTO || route > MD_ROUTE_PUSH || tile < 0) {
    set_error("bad plan, route %d or tile %lld", route, (long long)tile);
    return MD_ERR_INVALID_CONFIG;
  }
  p->route = route;
  p->tile = tile & ~int64_t(3);
  return MD_OK;
}

int md_plan_destroy(md_plan_t* p) {
  if (!p) return MD_OK;
  int prev;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  cudaFree(p->dev);
  cudaFree(p->prog_dev);
  cudaFree(p->owner_dev);
  cudaSetDevice(prev);
  delete p;
  return MD_OK;
}

}  // extern "C"

namespace {
using namespace md;

// Routing knobs, read ONCE per process (the environment is for tools and A/B
// runs; tests and callers pick routes per plan with md_plan_set_route).
struct ArEnv {
  int64_t ll_max = -1;       // MD_AR_LL_MAX: largest LL buffer (bytes), -1 = built-in
  int64_t oneshot_max = -1;  // MD_AR_ONESHOT_MAX
  int32_t route = MD_ROUTE_AUTO;  // MD_AR_ROUTE=tree|queue|ll|oneshot|stream|push
  int64_t tile = 0;          // MD_AR_TILE: tile of the tiled routes (elements)
  int32_t lag = -1;          // MD_AR_LAG: queue kernel pipeline lag
  bool trace = false;        // MD_AR_TRACE=1: per-CTA event log (md_trace_dump)
  bool sys_fence = false;    // MD_AR_SYS_FENCE=1: system-scope release for every flag
};

const ArEnv& ar_env() {
  static const ArEnv env = [] {
    ArEnv e;
    if (const char* x = getenv("MD_AR_LL_MAX")) e.ll_max = atoll(x);
    if (const char* x = getenv("MD_AR_ONESHOT_MAX")) e.oneshot_max = atoll(x);
    if (const char* x = getenv("MD_AR_TILE")) e.tile = std::max<int64_t>(0, atoll(x)) & ~int64_t(3);
    if (const char* x = getenv("MD_AR_LAG")) e.lag = std::max(0, atoi(x));
    e.trace = getenv("MD_AR_TRACE") != nullptr;
    e.sys_fence = getenv("MD_AR_SYS_FENCE") != nullptr;
    if (const char* x = getenv("MD_AR_ROUTE")) {
      static const char* names[] = {"auto", "tree", "queue", "ll", "oneshot", "stream", "push"};
      for (int r = 0; r <= MD_ROUTE_PUSH; ++r)
        if (!strcmp(x, names[r])) e.route = r;
    }
    return e;
  }();
  return env;
}

// Smallest plain buffer (bytes) the owner-push kernel takes by default.
// Measured against every other route (graph-timed C2 sweep, round 2,
// profiles/r02_sweep_n{2,4}.csv): N = 2 push 22.3 us at 4 MiB (one-shot 23.0)
// and 42.0 us at 16 MiB (tree 45.9-61.6), LL stays faster at 1 MiB (10.4 vs
// 17.9); N = 4 push 19.3 us at 1 MiB (LL 20.6-20.9) and faster at every size
// above.
int64_t push_min_bytes(int N) { return N == 2 ? (int64_t(4) << 20) : (int64_t(1) << 20); }

// Pipeline segment cap for a color chunk of `chunk` elements: about two
// segments per SM, never below 4096 elements (the per-segment flag cost).
// segment_elems is an upper bound only -- the bits never depend on it
// (pkg/tests/test_collectives.py:131-147). Measured at N = 4, k = 4: 4 MiB
// 38.3 -> 35.3 us, 16 MiB 65.9 -> 62 us; 100 MB unchanged (16384 stays).
int64_t auto_seg(int64_t chunk, int dev) {
  const int64_t want = (chunk / (2 * static_cast<int64_t>(sm_count(dev))) + 3) & ~int64_t(3);
  return std::max<int64_t>(4096, want);
}

// Largest buffer (bytes) the one-shot kernel takes at world size N: at N = 2
// its ingress equals the tree's, so any size that fits; above, it pulls
// (N-1) x bytes against the tree's 2 (N-1)/N x bytes, so only latency-bound
// sizes (measured crossover, profiles/README.md).
int64_t oneshot_max_bytes(int N) {
  if (ar_env().oneshot_max >= 0) return ar_env().oneshot_max;
  return N == 2 ? (int64_t(1) << 40) : (int64_t(1) << 20);
}

// Smallest buffer (bytes) a replicated fused N = 2 call streams (measured win
// at the 102.4 MB C5 buffer; below that the tree keeps it).
constexpr int64_t kStreamMinBytes = int64_t(64) << 20;

// Largest buffer (bytes) the LL push kernel takes: it moves 2 x (N-1) x bytes
// out of every rank (value + epoch words), so only latency-bound sizes:
// measured faster than the one-shot pull up to 1 MiB at N = 2 and 4 (10.4 vs
// 15.9 us and 20.0 vs 21.3 us), untested above N = 4 (256 KiB there).
int64_t ll_max_bytes(int N) {
  if (ar_env().ll_max >= 0) return ar_env().ll_max;
  return N <= 4 ? (int64_t(1) << 20) : (int64_t(256) << 10);
}

// diagnostics (MD_AR_TRACE=1): the per-CTA event log of this call, one per device
int setup_trace(AllreduceArgs* a, int dev, int ctas, int n_views) {
  a->trace = nullptr;
  if (!ar_env().trace || dev < 0 || dev >= 64) return MD_OK;
  const size_t bytes = sizeof(TraceEv) * 3 * kTraceHalf * static_cast<size_t>(ctas) * n_views;
  if (!g_trace[dev].ptr || g_trace[dev].bytes < bytes) {
    if (g_trace[dev].ptr) cudaFree(g_trace[dev].ptr);
    MD_CUDA_TRY(cudaMalloc(&g_trace[dev].ptr, bytes));
    MD_CUDA_TRY(cudaMemset(g_trace[dev].ptr, 0, bytes));
    g_trace[dev].bytes = bytes;
  }
  // (md_trace_dump re-zeroes the log, so a traced call adds no work of its own)
  g_trace[dev].used = bytes;
  a->trace = static_cast<TraceEv*>(g_trace[dev].ptr);
  return MD_OK;
}

// cudaFuncSetAttribute(max dynamic SMEM) once per (kernel, device)
int smem_attr_once(const void* k, int dev, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  std::lock_guard<std::mutex> g(mu);
  for (const auto& d : done)
    if (d.first == k && d.second == dev) return MD_OK;
  MD_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(bytes)));
  done.emplace_back(k, dev);
  return MD_OK;
}

// Emulated ranks (n_views > 1) wait on each other's CTAs on ONE device: a
// cooperative launch guarantees they are co-resident. A real rank's CTAs only
// wait on other GPUs (never on a sibling CTA), so a plain launch of <= one
// CTA per SM is deadlock-free there.
int launch_views(const void* k, unsigned grid, int n_views, size_t smem, AllreduceArgs* a,
                 void* stream, int threads = kArThreads) {
  void* args[] = {a};
  if (n_views > 1) {
    MD_CUDA_TRY(cudaLaunchCooperativeKernel(k, dim3(grid * n_views), dim3(threads), args, smem,
                                            as_stream(stream)));
  } else {
    MD_CUDA_TRY(cudaLaunchKernel(k, dim3(grid), dim3(threads), args, smem, as_stream(stream)));
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return MD_OK;
}


std::atomic<uint64_t> g_last_route[64];

void record_route(int dev, int route, int64_t tile, bool sharded) {
  if (dev >= 0 && dev < 64)
    g_last_route[dev].store(static_cast<uint64_t>(route) | (sharded ? 0x80u : 0u) |
                                (static_cast<uint64_t>(tile) << 8),
                            std::memory_order_relaxed);
}

uint64_t cfg_word_of(int route, bool owner_sched, bool sharded, int64_t geometry) {
  return static_cast<uint64_t>(route) | (static_cast<uint64_t>(owner_sched) << 4) |
         (static_cast<uint64_t>(sharded) << 5) | (static_cast<uint64_t>(geometry) << 8);
}

}  // namespace

extern "C" {

int md_last_route(int32_t device, int32_t* route, int64_t* tile, int32_t* sharded) {
  if (device < 0 || device >= 64) {
    set_error("bad device %d", device);
    return MD_ERR_INVALID_CONFIG;
  }
  const uint64_t w = g_last_route[device].load(std::memory_order_relaxed);
  if (route) *route = static_cast<int32_t>(w & 0x7f);
  if (sharded) *sharded = (w & 0x80) ? 1 : 0;
  if (tile) *tile = static_cast<int64_t>(w >> 8);
  return MD_OK;
}

int md_allreduce(md_comm_t* const* comms, int32_t n_views, const md_plan_t* plan,
                 float* const* bufs, int64_t n, const float* const* workers, int32_t n_workers,
                 float* const* w, float* const* mom, int64_t update_len, float c, float mu,
                 float wd_b, int64_t seg_elems, int32_t ctas, void* stream) {
  md_update_t u{w, mom, update_len, c, mu, wd_b, MD_UPDATE_REPLICATED};
  return md_allreduce_ex(comms, n_views, plan, bufs, n, workers, n_workers, w ? &u : nullptr,
                         seg_elems, ctas, stream);
}

int md_allreduce_ex(md_comm_t* const* comms, int32_t n_views, const md_plan_t* plan,
                    float* const* bufs, int64_t n, const float* const* workers, int32_t n_workers,
                    const md_update_t* upd, int64_t seg_elems, int32_t ctas, void* stream) {
  if (!plan || n_views < 1 || n_views > MD_MAX_RANKS) {
    set_error("bad plan/view count");
    return MD_ERR_INVALID_CONFIG;
  }
  const int N = plan->n_ranks;
  const ArEnv& env = ar_env();
  if (n < 0) {
    set_error("negative length");
    return MD_ERR_INVALID_CONFIG;
  }
  if (n_workers < 0 || n_workers > MD_MAX_WORKERS || (n_workers > 0 && !workers)) {
    set_error("bad worker count %d (max %d)", n_workers, MD_MAX_WORKERS);
    return MD_ERR_INVALID_CONFIG;
  }
  if (seg_elems < 1) {
    set_error("segment_elems must be >= 1, got %lld", (long long)seg_elems);
    return MD_ERR_INVALID_CONFIG;
  }
  const bool has_update = upd != nullptr && upd->w != nullptr;
  const int64_t update_len = has_update ? upd->len : 0;
  if (has_update && (update_len < 0 || update_len > n)) {
    set_error("update_len %lld outside [0, %lld]", (long long)update_len, (long long)n);
    return MD_ERR_LENGTH_MISMATCH;
  }
  if (has_update && upd->mode != MD_UPDATE_REPLICATED && upd->mode != MD_UPDATE_SHARDED) {
    set_error("bad update mode %d", upd->mode);
    return MD_ERR_INVALID_CONFIG;
  }
  const bool mode_sharded = has_update && upd->mode == MD_UPDATE_SHARDED;
  const float c = has_update ? upd->c : 0.f, mu = has_update ? upd->mu : 0.f;
  const float wd_b = has_update ? upd->wd_b : 0.f;
  int dev;
  MD_CUDA_TRY(cudaGetDevice(&dev));
  AllreduceArgs a;
  memset(&a, 0, sizeof(a));
  a.plan = plan->dev;
  a.n = n;
  a.n_ranks = N;
  a.k = plan->k;
  a.n_views = n_views;
  a.n_workers = n_workers;
  a.has_update = has_update;
  a.update_len = update_len;
  a.c = c;
  a.mu = mu;
  a.wd_b = wd_b;
  a.flag_gpu_fence = !env.sys_fence;  // see publish_flags
  a.reverse_local = 1;
  a.prog = plan->prog_dev;
  a.prog_k = plan->k;
  // segment length: multiple of 4 elements, <= kMaxSegs segments per color
  const int64_t maxlen = (n + plan->k - 1) / plan->k;
  int64_t seg = std::max<int64_t>(4, (seg_elems + 3) & ~int64_t(3));
  if (N > 1) seg = std::min(seg, auto_seg(maxlen, dev));
  const int64_t min_seg = ((maxlen + 3) / kMaxSegs + 4 + 3) & ~int64_t(3);
  if (seg < min_seg) seg = min_seg;
  a.seg = seg;
  int64_t mx = 0;
  for (int col = 0; col < plan->k; ++col) {
    int64_t st, ln;
    chunk_of(n, plan->k, col, &st, &ln);
    mx = std::max(mx, nseg_of(st, ln, seg));
  }
  a.max_nseg = static_cast<int32_t>(mx);
  uintptr_t bits = 0;
  double timeout = 30.0;
  for (int vi = 0; vi < n_views; ++vi) {
    md_comm* cm = comms[vi];
    if (!cm || cm->n_ranks != N) {
      set_error("communicator/plan world size mismatch (%d vs %d)", cm ? cm->n_ranks : -1, N);
      return MD_ERR_INVALID_CONFIG;
    }
    ViewArgs& v = a.v[vi];
    v.rank = cm->rank;
    v.ctrl = cm->ctrl;
    for (int r = 0; r < N; ++r) {
      if (!cm->peer_ctrl[r]) {
        set_error("rank %d: control block of peer %d not installed", cm->rank, r);
        return MD_ERR_INVALID_CONFIG;
      }
      v.peer_ctrl[r] = cm->peer_ctrl[r];
      v.peer[r] = bufs[vi * N + r];
      bits |= reinterpret_cast<uintptr_t>(v.peer[r]);
    }
    v.buf = bufs[vi * N + cm->rank];
    for (int j = 0; j < n_workers; ++j) {
      v.workers[j] = workers[vi * n_workers + j];
      bits |= reinterpret_cast<uintptr_t>(v.workers[j]);
    }
    if (has_update) {
      // sharded: w holds every rank's (peer-mapped) weights, view-major
      v.w = mode_sharded ? upd->w[vi * N + cm->rank] : upd->w[vi];
      if (mode_sharded)
        for (int r = 0; r < N; ++r) {
          v.peer_w[r] = upd->w[vi * N + r];
          bits |= reinterpret_cast<uintptr_t>(v.peer_w[r]);
        }
      v.mom = (upd->mom && mu != 0.f) ? upd->mom[vi] : nullptr;
      bits |= reinterpret_cast<uintptr_t>(v.w) | reinterpret_cast<uintptr_t>(v.mom);
    }
    v.err = cm->err_dev;
    ++cm->epoch;
    timeout = std::min(timeout, cm->timeout_s);
  }
  a.vec_ok = (bits & 15) == 0;
  a.timeout_ns = static_cast<unsigned long long>(timeout * 1e9);
  const int req = plan->route != MD_ROUTE_AUTO ? plan->route : env.route;
  const int64_t tile_req = plan->tile ? plan->tile : env.tile;
  const bool auto_route = req == MD_ROUTE_AUTO;
  const int avail = sm_count(dev) / n_views;  // CTAs (one per SM) per view
  const bool fold_ok = N > 1 && n > 0 && n_workers == 0 && a.vec_ok && plan->prog_dev;

  // One rank, no worker fold: the collective is the identity and the call is
  // only its fused SGD update -- the streaming md_sgd_update kernel (8 CTAs x
  // 256 threads per SM) measured 82 vs 91 us for the 25.6M-float momentum +
  // weight-decay update (95 % vs 86 % of the HBM copy peak); same sgd1 math.
  if (N == 1 && n_views == 1 && n_workers == 0) {
    record_route(dev, MD_ROUTE_LOCAL, 0, false);
    if (!has_update || update_len == 0) return MD_OK;
    return md_sgd_update(a.v[0].w, a.v[0].buf, a.v[0].mom, update_len, c,
                         a.v[0].mom ? mu : 0.f, wd_b, stream);
  }
  int epi = 0;
  if (has_update) epi = (a.v[0].mom ? 3 : 1) + (wd_b != 0.f ? 1 : 0);

  // ---- owner-push: plain buffers from push_min_bytes(N), and every sharded
  // update (W' pushed, momentum sharded; see allreduce_push_kernel)
  {
    const bool shard_ok = mode_sharded && (update_len & 3) == 0;
    const bool want = shard_ok ? (auto_route || req == MD_ROUTE_PUSH)
                               : epi == 0 && (req == MD_ROUTE_PUSH ||
                                              (auto_route && n * 4 >= push_min_bytes(N)));
    if (want && fold_ok && avail >= 1) {
      // tile: deep enough rings for the N sources (measured, graph-timed 1 GiB:
      // N = 4 2048 -> 2361 us vs 4096 -> 2596 us; N = 2 3072 -> 1615 vs 1636)
      int64_t TE = tile_req ? tile_req : (N == 2 ? 3072 : 2048);
      int64_t A0, B0;
      push_slice(n, N, 0, &A0, &B0);
      if (!tile_req) {  // balanced: every CTA gets the same number of tiles (no ragged last wave)
        const int64_t rounds = std::max<int64_t>(1, (B0 - A0 + avail * TE - 1) / (avail * TE));
        TE = std::max<int64_t>(4, ((B0 - A0 + avail * rounds - 1) / (avail * rounds) + 3) &
                                      ~int64_t(3));
      }
      while ((B0 - A0 + TE - 1) / TE > kMaxTiles) TE *= 2;
      const int ups = epi == 0 ? 0 : (epi >= 3 ? 2 : 1);
      const int64_t stage_bytes = static_cast<int64_t>(N + 1 + ups) * TE * 4;
      // ring: the 192 KB of round 1 for plain calls (measured: a 6th stage from
      // the 224 KB ring made 1 GiB at N = 2 3 % slower), 224 KB when the W /
      // momentum rows ride along (sharded update)
      const int64_t ring = epi == 0 ? kRingBytes : kStreamRingBytes;
      const int S = static_cast<int>(std::min<int64_t>(8, ring / stage_bytes));
      if (S >= 2) {
        const int64_t T = std::max<int64_t>(1, (B0 - A0 + TE - 1) / TE);
        const int g = static_cast<int>(std::min<int64_t>(avail, T));
        a.seg = TE;
        a.lag = S;
        a.ctas_per_view = g;
        a.sharded = shard_ok;
        a.exit_sys_release = 1;
        a.cfg_word = cfg_word_of(MD_ROUTE_PUSH, false, shard_ok, TE);
        const void* k = allreduce_push_kernel_of(epi);
        const size_t smem = static_cast<size_t>(S) * stage_bytes;
        int rc = smem_attr_once(k, dev, kStreamRingBytes);
        if (rc == MD_OK) rc = setup_trace(&a, dev, g, n_views);
        if (rc == MD_OK) rc = launch_views(k, g, n_views, smem, &a, stream);
        if (rc == MD_OK) record_route(dev, MD_ROUTE_PUSH, TE, shard_ok);
        return rc;
      }
    }
  }

  // ---- LL push (the smallest buffers): see allreduce_ll_kernel
  {
    const int64_t g0 = std::min<int64_t>(avail, std::max<int64_t>(1, (n + 255) / 256));
    const int64_t E = g0 > 0 ? (((n + g0 - 1) / g0) + 3) & ~int64_t(3) : 0;
    const bool want = req == MD_ROUTE_LL || (auto_route && n * 4 <= ll_max_bytes(N));
    if (want && fold_ok && n <= kLLElems && avail >= 1 && N * E * 4 <= int64_t(kRingBytes)) {
      const int64_t g = (n + E - 1) / E;
      a.seg = E;
      a.ctas_per_view = static_cast<int32_t>(g);
      const void* k = allreduce_ll_kernel_of(epi);
      int rc = smem_attr_once(k, dev, kRingBytes);
      if (rc == MD_OK)
        rc = launch_views(k, static_cast<unsigned>(g), n_views, static_cast<size_t>(N) * E * 4,
                          &a, stream);
      if (rc == MD_OK) record_route(dev, MD_ROUTE_LL, E, false);
      return rc;
    }
  }

  // ---- one-shot pull (buffers that fit one SMEM pass of every rank's data)
  {
    const int64_t emax = static_cast<int64_t>(kRingBytes / 4u / N) & ~int64_t(3);
    int64_t g = std::min<int64_t>(avail, std::max<int64_t>(1, (n + 1023) / 1024));
    const int64_t E = (((n + g - 1) / g) + 3) & ~int64_t(3);
    const bool want = req == MD_ROUTE_ONESHOT || (auto_route && n * 4 <= oneshot_max_bytes(N));
    if (want && fold_ok && avail >= 1 && E <= emax) {
      g = (n + E - 1) / E;
      a.seg = E;
      a.ctas_per_view = static_cast<int32_t>(g);
      a.cfg_word = cfg_word_of(MD_ROUTE_ONESHOT, false, false, E);
      const void* k = allreduce_oneshot_kernel_of(epi);
      int rc = smem_attr_once(k, dev, kRingBytes);
      if (rc == MD_OK)
        rc = launch_views(k, static_cast<unsigned>(g), n_views, static_cast<size_t>(N) * E * 4,
                          &a, stream);
      if (rc == MD_OK) record_route(dev, MD_ROUTE_ONESHOT, E, false);
      return rc;
    }
  }

  // ---- stream (all-pull, tiled): replicated fused calls at N = 2 from 64 MiB,
  // balanced tiles of <= 6656 floats (two stages of [2 ranks | W | momentum]
  // in the 224 KB ring): C5 step at N = 2, graph-timed, 206 -> 198 us
  // (profiles/README.md). At N > 2 it pulls (N-1) x bytes and loses (N = 4:
  // 502 vs 275 us), so there it only runs when asked for.
  {
    const bool want =
        req == MD_ROUTE_STREAM || (auto_route && N == 2 && epi != 0 && n * 4 >= kStreamMinBytes);
    if (want && fold_ok && avail >= 1) {
      int64_t TE = 2048;
      if (N == 2) {  // balanced: every CTA gets the same number of tiles
        const int64_t rounds = std::max<int64_t>(1, (n + avail * 6656 - 1) / (avail * 6656));
        TE = std::max<int64_t>(4, ((n + avail * rounds - 1) / (avail * rounds) + 3) & ~int64_t(3));
      }
      if (tile_req) TE = tile_req;
      while ((n + TE - 1) / TE > kMaxTiles) TE *= 2;
      const int epi_slots = epi == 0 ? 0 : (epi >= 3 ? 2 : 1);
      const int64_t stage_bytes = static_cast<int64_t>(N + epi_slots) * TE * 4;
      const int S = static_cast<int>(std::min<int64_t>(8, kStreamRingBytes / stage_bytes));
      if (S >= 2) {
        const int64_t T = (n + TE - 1) / TE;
        const int g = static_cast<int>(std::min<int64_t>(avail, T));
        a.seg = TE;
        a.lag = S;
        a.ctas_per_view = g;
        a.cfg_word = cfg_word_of(MD_ROUTE_STREAM, false, false, TE);
        const void* k = allreduce_stream_kernel_of(epi);
        int rc = smem_attr_once(k, dev, kStreamRingBytes);
        if (rc == MD_OK)
          rc = launch_views(k, g, n_views, static_cast<size_t>(S) * stage_bytes, &a, stream);
        if (rc == MD_OK) record_route(dev, MD_ROUTE_STREAM, TE, false);
        return rc;
      }
    }
  }

  // ---- the pipelined tree: every other call (fused updates at N > 2, worker
  // folds, unaligned buffers). The owner-computes schedule
  // (md_plan_set_schedule, build_owner_plans) runs the same channelized
  // kernel over the owner plan (n slices), each owner evaluating the plan's
  // fold programs; worker folds and unaligned buffers keep the tree schedule
  // (same bits either way).
  auto weighted_of = [&](const std::vector<RankPlan>& plans) {
    int wmax = 0;
    for (const RankPlan& rp : plans) {
      int wt = 0;
      for (int i = 0; i < rp.n_tasks; ++i) {
        const Task& t = rp.t[i];
        wt += t.type == 1 || t.n_fold > 1 || t.parent < 0 || n_workers > 0;
      }
      wmax = std::max(wmax, wt);
    }
    return wmax;
  };
  // (the owner plan needs the channelized kernel: one CTA per task at least)
  const bool owner = plan->schedule == MD_SCHED_OWNER && N > 1 && n_workers == 0 && a.vec_ok &&
                     req != MD_ROUTE_QUEUE && plan->owner_dev && plan->prog_dev &&
                     weighted_of(plan->owner_host) <= avail;
  const std::vector<RankPlan>& hp = owner ? plan->owner_host : plan->host;
  if (owner) {
    a.plan = plan->owner_dev;
    a.k = N;
    const int64_t ml = (n + N - 1) / N;
    const int64_t sg =
        std::min(std::max<int64_t>(4, (seg_elems + 3) & ~int64_t(3)), auto_seg(ml, dev));
    const int64_t ms = ((ml + 3) / kMaxSegs + 4 + 3) & ~int64_t(3);
    a.seg = std::max(sg, ms);
    int64_t mx2 = 0;
    for (int col = 0; col < N; ++col) {
      int64_t st, ln;
      chunk_of(n, N, col, &st, &ln);
      mx2 = std::max(mx2, nseg_of(st, ln, a.seg));
    }
    a.max_nseg = static_cast<int32_t>(mx2);
  }
  // 16-byte aligned buffers take the channelized TMA kernel; anything else
  // the work-queue kernel with its scalar path (MD_ROUTE_QUEUE forces it)
  // (and only when every task of every rank can own at least one CTA)
  const bool chan = a.vec_ok && req != MD_ROUTE_QUEUE && weighted_of(hp) <= avail;
  const void* kern = chan ? allreduce_channels_kernel_of(epi) : allreduce_kernel_of(epi);
  int rc = smem_attr_once(kern, dev, kRingBytes);
  if (rc != MD_OK) return rc;
  int per_sm = 0;
  const int threads = chan ? kChanThreads : kArThreads;
  MD_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads,
                                                             kRingBytes));
  const int resident = per_sm * sm_count(dev);
  if (ctas <= 0) ctas = resident / n_views;
  ctas = std::min(ctas, resident / n_views);
  if (ctas < 1) {
    set_error("%d views do not fit co-resident on device %d", n_views, dev);
    return MD_ERR_INVALID_CONFIG;
  }
  a.ctas_per_view = ctas;
  // lag: about one CTA wave of items per pipeline stage (override: MD_AR_LAG)
  int max_stage = 0, max_tasks = 1;
  for (const RankPlan& rp : hp) {
    max_tasks = std::max(max_tasks, rp.n_tasks);
    for (int i = 0; i < rp.n_tasks; ++i) max_stage = std::max(max_stage, rp.t[i].stage);
  }
  a.lag = env.lag >= 0 ? env.lag : std::max(1, ctas / max_tasks);
  a.max_stage = max_stage;
  // the queue and channelized kernels exchange the same per-segment flags
  a.cfg_word = cfg_word_of(MD_ROUTE_TREE, owner, false, a.seg);
  rc = setup_trace(&a, dev, ctas, n_views);
  if (rc == MD_OK) rc = launch_views(kern, ctas, n_views, kRingBytes, &a, stream, threads);
  if (rc == MD_OK) record_route(dev, chan ? MD_ROUTE_TREE : MD_ROUTE_QUEUE, a.seg, false);
  return rc;
}

}  // extern "C"

extern "C" int md_trace_dump(int32_t device, const char* path) {
  if (device < 0 || device >= 64 || !g_trace[device].ptr) {
    set_error("no allreduce trace on device %d (set MD_AR_TRACE=1)", device);
    return MD_ERR_INVALID_CONFIG;
  }
  std::vector<char> host(g_trace[device].used);
  int prev;
  MD_CUDA_TRY(cudaGetDevice(&prev));
  MD_CUDA_TRY(cudaSetDevice(device));
  cudaError_t e = cudaMemcpy(host.data(), g_trace[device].ptr, host.size(), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemset(g_trace[device].ptr, 0, g_trace[device].bytes);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    set_error("trace copy: %s", cudaGetErrorString(e));
    return MD_ERR_CUDA;
  }
  FILE* f = fopen(path, "wb");
  if (!f) {
    set_error("cannot write %s", path);
    return MD_ERR_INVALID_CONFIG;
  }
  fwrite(host.data(), 1, host.size(), f);
  fclose(f);
  return MD_OK;
}
