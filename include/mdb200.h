/*
 * mdb200.h -- C ABI of libmdb200.so, the B200 (sm_100a) data-parallel hot path
 * of arXiv 1711.00705 as re-created by the reference package `minidist`.
 *
 * Every entry point takes plain pointers, sizes and an opaque CUDA stream
 * (`void* stream`, a cudaStream_t; NULL = legacy default stream). No torch
 * types cross this boundary. Return value: MD_OK (0) or a negative MD_ERR_*
 * code; md_last_error() returns a thread-local message for the last failure.
 * The Python host layer maps codes onto the reference's exception classes
 * (/root/reference/pkg/src/minidist/errors.py:4-65).
 *
 * Each declaration names the reference interface it replaces (file:line,
 * relative to /root/reference/pkg/src/minidist/).
 */
#ifndef MDB200_H
#define MDB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes --------------------------------------------------------- */
#define MD_OK 0
#define MD_ERR_LENGTH_MISMATCH (-1) /* ValueError / LengthMismatch (errors.py:16) */
#define MD_ERR_INVALID_CONFIG (-2)  /* InvalidConfig (errors.py:8)                */
#define MD_ERR_CUDA (-3)            /* CUDA runtime failure                        */
#define MD_ERR_TIMEOUT (-4)         /* NotExposed: a peer never signalled (errors.py:32) */
#define MD_ERR_OFFSET_OVERFLOW (-5) /* OffsetOverflow (errors.py:20)               */
#define MD_ERR_EMPTY_SHARD (-6)     /* EmptyShard (errors.py:52)                   */
#define MD_ERR_DIVERGENCE (-7)      /* DivergenceDetected (errors.py:60)           */

#define MD_MAX_RANKS 16   /* largest world (or emulated world) a plan supports */
#define MD_MAX_COLORS 16  /* k colors per tree set                             */
#define MD_MAX_WORKERS 8  /* worker buffers folded by the fused prologue       */
#define MD_MAX_GROUP 64   /* DIMD group size                                   */
#define MD_IPC_HANDLE_BYTES 64

const char* md_last_error(void);
/* Library/ABI version; bumps when a signature changes. */
int md_version(void);
/* Number of kernel launches this process made through the library (all
 * entry points). bench.py reads it to report `gpu_launches`. */
uint64_t md_launch_count(void);

/* ---- operator seam: minidist._kernels ----------------------------------- */
/* dst[i] += src[i] (f32, round-to-nearest, no contraction).
 * Replaces add_f32, _kernels/_accel.pyx:12-19 (numpy twin fallback.py:6-12).
 * n_dst != n_src -> MD_ERR_LENGTH_MISMATCH (the reference's ValueError). */
int md_add_f32(float* dst, int64_t n_dst, const float* src, int64_t n_src, void* stream);

/* dst[i] = dst[i] - fl32(fl32(c) * src[i]): two roundings, never an FMA.
 * Replaces sub_scaled_f32, _kernels/_accel.pyx:22-29 (fallback.py:15-23). */
int md_sub_scaled_f32(float* dst, int64_t n_dst, const float* src, int64_t n_src, double c,
                      void* stream);

/* Momentum / weight-decay extension of the update at sgd.py:416 (the
 * reference has plain SGD; this is NOT in the reference):
 *   d = g                        (+ fl(wd_b * w)   if wd_b != 0)
 *   v = fl(fl(mu * v) + d); d = v                 (if mom != NULL)
 *   w = fl(w - fl(c * d))
 * With mom == NULL and wd_b == 0 it is bit-identical to md_sub_scaled_f32. */
int md_sgd_update(float* w, const float* g, float* mom, int64_t n, float c, float mu, float wd_b,
                  void* stream);

/* Deterministic per-rank fill of the reference benchmark,
 * bench.py:188-195: buf[i] = f32(((i mod 997) + 1) * (rank + 1) * pi / n_ranks). */
int md_fill_rank_input(float* buf, int64_t n, int32_t rank, int32_t n_ranks, void* stream);

/* ---- peer memory (the transport's expose/pull, transport/base.py:191-240) -- */
/* Export the allocation that contains `ptr` (cudaMalloc / torch caching
 * allocator memory) as a CUDA IPC handle; *offset = ptr - allocation base. */
int md_mem_export(const void* ptr, unsigned char handle[MD_IPC_HANDLE_BYTES], uint64_t* offset);
/* Map a peer process's allocation; *base receives the mapped base address. */
int md_mem_import(const unsigned char handle[MD_IPC_HANDLE_BYTES], void** base);
int md_mem_close(void* base);
/* In-process multi-GPU: enable direct loads/stores from `dev` into `peer`. */
int md_enable_peer_access(int dev, int peer);
int md_device_count(int* n);

/* ---- communicator (one per rank; the endpoint of transport/runner.py:29) -- */
typedef struct md_comm md_comm_t;
/* Allocates this rank's control block (flags for the epoch protocol) on
 * `device` and a host-mapped error word. */
int md_comm_create(int32_t rank, int32_t n_ranks, int32_t device, md_comm_t** out);
int md_comm_destroy(md_comm_t* comm);
/* Control block pointer/handle, for the host-side handle exchange. */
int md_comm_ctrl_ptr(md_comm_t* comm, void** ctrl);
/* Install every rank's control block as seen from this process (index =
 * rank; the own entry is ignored). Multi-process callers pass imported
 * pointers, in-process callers pass the peers' md_comm_ctrl_ptr values. */
int md_comm_set_peer_ctrl(md_comm_t* comm, void* const* ctrl_ptrs, int32_t n);
/* Error word written by device code (MD_ERR_* or 0); reading it resets it.
 * Only meaningful after the stream that ran the collective synchronized. */
int md_comm_take_error(md_comm_t* comm, int32_t* code, int32_t* detail);
/* Watchdog for device-side flag waits (seconds; reference default 30 s,
 * transport/base.py:28). */
int md_comm_set_timeout(md_comm_t* comm, double seconds);

/* ---- fold plans: topology.py:132-173 (multicolor), :123-129 (ring) --------- */
typedef struct md_plan md_plan_t;
/* One fold tree per color. For color c and rank r (row c*n_ranks + r):
 *   parent[.]  = parent rank or -1 at the root (exactly one root per color);
 *   children   = child_idx[child_ptr[.] .. child_ptr[. + 1]) in fold order;
 *   self_pos   = where the node's own value enters its fold (NULL = 0 for every
 *                node: "own value, then children in child-list order",
 *                collectives.py:271-286). reduce_then_broadcast's rank-order
 *                root fold (collectives.py:384-399) is a star whose root has
 *                self_pos = its rank.
 * child_ptr has k*n_ranks + 1 entries (CSR over all rows). */
int md_plan_create(int32_t n_ranks, int32_t k, const int32_t* parent, const int32_t* child_ptr,
                   const int32_t* child_idx, const int32_t* self_pos, int32_t device,
                   md_plan_t** out);
int md_plan_destroy(md_plan_t* plan);
/* Data movement of md_allreduce for this plan (never changes the bits):
 * MD_SCHED_TREE (default) reduces and broadcasts each color along its own
 * tree (collectives.py:225-296); MD_SCHED_OWNER cuts the buffer into n_ranks
 * slices, rank j pulls slice j from every rank and evaluates each element's
 * color fold in the tree's order, then every rank copies the final slices --
 * 2 (n-1)/n of the buffer in per rank for any k. */
#define MD_SCHED_TREE 0
#define MD_SCHED_OWNER 1
int md_plan_set_schedule(md_plan_t* plan, int32_t schedule);

/* Kernel route of md_allreduce for this plan (never changes the bits; see
 * md_allreduce for what each one does). MD_ROUTE_AUTO picks by size, world
 * size and update mode; any other value forces that route where it applies
 * (a route that cannot serve a call -- e.g. LL with a worker fold, owner-push
 * with a replicated update -- falls back to MD_ROUTE_TREE).
 * tile: elements per tile of the tiled routes (stream, push); 0 = auto.
 * The environment variable MD_AR_ROUTE=tree|queue|ll|oneshot|stream|push
 * (read once per process) sets the default for plans left on AUTO. */
#define MD_ROUTE_AUTO 0
#define MD_ROUTE_TREE 1    /* channelized pipelined tree (or owner plan)     */
#define MD_ROUTE_QUEUE 2   /* work-queue tree kernel (scalar path, any alignment) */
#define MD_ROUTE_LL 3      /* LL push                                         */
#define MD_ROUTE_ONESHOT 4 /* one-shot pull                                   */
#define MD_ROUTE_STREAM 5  /* tiled all-pull with per-tile read-done flags    */
#define MD_ROUTE_PUSH 6    /* owner-push (plain calls and sharded updates)    */
#define MD_ROUTE_LOCAL 7   /* (reported only) N = 1: update kernel alone      */
int md_plan_set_route(md_plan_t* plan, int32_t route, int64_t tile);
/* Route (MD_ROUTE_*), tile/segment and update mode (1 = sharded) of the
 * last md_allreduce launched on `device` by this process. */
int md_last_route(int32_t device, int32_t* route, int64_t* tile, int32_t* sharded);

/* ---- allreduce: collectives.py:225-296 (multicolor), :302-359 (ring),
 *      :365-409 (reduce_then_broadcast); dispatcher :412-429 ----------------- */
/* One persistent kernel per call. `n_views` ranks are served by this call:
 * 1 for a real rank (one GPU per rank), n_ranks when every rank of the
 * world is emulated on one GPU (then comms[v] is rank v's communicator).
 * The kernel is picked by size (md_plan_set_route overrides); all of them
 * produce the same bits (the plan's fold order per color), which the GPU
 * tests check for every path:
 *   LL push      n*4 <= 1 MiB (N <= 4; 256 KiB above): every rank pushes
 *                (value, epoch) words into its peers' control-block inbox and
 *                folds locally -- one NVLink trip, no barrier (MD_AR_LL_MAX);
 *   one-shot     N = 2 between the LL and owner-push ranges (up to one SMEM
 *                pass of every rank's data, ~14 MB, when pinned): pull every
 *                peer buffer, fold locally (MD_AR_ONESHOT_MAX);
 *   owner-push   plain buffers (no fused update / worker fold) from 4 MiB at
 *                N = 2, 1 MiB above, and every SHARDED update
 *                (md_allreduce_ex): rank j pulls slice j of every rank,
 *                folds it with each element's color program and TMA-stores
 *                the result (or, sharded, the updated weights) into every
 *                rank's buffer;
 *   stream       replicated fused SGD updates at N = 2 from 64 MiB: tiled
 *                all-pull through a TMA ring with per-tile read-done flags,
 *                balanced <= 6656-float tiles (C5 step 206 -> 198 us);
 *   tree         everything else (fused updates, worker folds, unaligned
 *                buffers): the pipelined per-color reduce + broadcast over
 *                peer memory (or the owner plan, md_plan_set_schedule).
 *
 *   bufs      [n_views * n_ranks]: for view v, rank r's gradient buffer as
 *             addressable from this process (peer-mapped); bufs[v*n+rank(v)]
 *             is the view's own buffer, updated in place.
 *   n         elements per buffer (every rank must pass the same n, else all
 *             ranks fail with MD_ERR_LENGTH_MISMATCH -- _check_same_length,
 *             collectives.py:157-174).
 *   workers   [n_views * n_workers] or NULL: fused gradient accumulation --
 *             the own value is fold(workers) in worker order (sgd.py:335-353)
 *             instead of the buffer's contents.
 *   w, mom    [n_views] or NULL: fused SGD epilogue (md_sgd_update semantics)
 *             on the first update_len elements once the sum is final.
 *   seg_elems pipeline granularity (elements); results do not depend on it
 *             (pkg/tests/test_collectives.py:131-147).
 *   ctas      CTAs per view (0 = auto).
 * Every rank must take the same route with the same geometry; the entry
 * barrier compares a route word across ranks and fails every rank with
 * MD_ERR_INVALID_CONFIG if they differ (e.g. one rank's buffers misaligned). */
int md_allreduce(md_comm_t* const* comms, int32_t n_views, const md_plan_t* plan,
                 float* const* bufs, int64_t n, const float* const* workers, int32_t n_workers,
                 float* const* w, float* const* mom, int64_t update_len, float c, float mu,
                 float wd_b, int64_t seg_elems, int32_t ctas, void* stream);

/* Fused SGD epilogue of md_allreduce_ex (md_sgd_update semantics on the
 * first `len` elements once the sum is final).
 *   MD_UPDATE_REPLICATED: w, mom are [n_views]; every rank updates its full
 *     replica (the reference's replicated weights, sgd.py:416).
 *   MD_UPDATE_SHARDED: w is [n_views * n_ranks] (view v, rank r: rank r's
 *     weights as addressable from this process -- peer-mapped), mom is
 *     [n_views]. The owner of each buffer slice updates it and pushes the
 *     new weights into every rank (same bits: replicas are identical,
 *     sgd.py:5-10); momentum is sharded state (only the own slice is read and
 *     written) and the buffer holds the sum only on the own slice and past
 *     `len`. Needs n_ranks > 1, no worker fold, 16-byte aligned buffers and
 *     len % 4 == 0; otherwise the call runs replicated (a superset: same
 *     weights, full sum, full momentum). */
#define MD_UPDATE_REPLICATED 0
#define MD_UPDATE_SHARDED 1
typedef struct md_update {
  float* const* w;
  float* const* mom;
  int64_t len;
  float c, mu, wd_b;
  int32_t mode;
} md_update_t;
int md_allreduce_ex(md_comm_t* const* comms, int32_t n_views, const md_plan_t* plan,
                    float* const* bufs, int64_t n, const float* const* workers, int32_t n_workers,
                    const md_update_t* update, int64_t seg_elems, int32_t ctas, void* stream);

/* Diagnostics: with MD_AR_TRACE=1 in the environment every md_allreduce
 * records %globaltimer events per CTA (flag waits, chunk arrival, segment
 * completion, publish); this writes the last call's log on `device` to
 * `path` (records of {u64 t_ns, u32 cta, u16 event, u16 segment}). */
int md_trace_dump(int32_t device, const char* path);

/* ---- DIMD store: dimd.py ------------------------------------------------- */
/* _mix64, dimd.py:226-234 (host, pure). */
uint64_t md_mix64(const uint64_t* parts, int32_t n);

/* random_batch, dimd.py:213-220: picks[i] = Philox(key).integers(0, n_records, batch)[i]
 * (numpy Philox4x64-10 stream, 32-bit Lemire with rejection). Device output. */
int md_random_batch(uint64_t key, int64_t n_records, int64_t batch, int64_t* picks, void* stream);

/* Diagnostics: a one-thread kernel that writes %globaltimer (ns) to *dst when
 * it runs on `stream` (brackets a call on the device's own clock). */
int md_stamp(uint64_t* dst, void* stream);

/* Graph-replayable random_batch for a training loop: the key is
 * _mix64(seed, role, worker, *step) computed on device (sgd.py:303-307) and
 * *step (device int64) is incremented by the kernel, so a captured CUDA graph
 * draws the next step's batch on every replay. batch <= 1024. */
int md_random_batch_step(uint64_t seed, uint64_t role, uint64_t worker, int64_t* step,
                         int64_t n_records, int64_t batch, int64_t* picks, void* stream);

/* Gather records picks[0..batch) of a shard (blob + index off/len/label) into
 * `out`: fixed stride when out_stride > 0 (every picked record must be exactly
 * out_stride bytes, else MD_ERR_LENGTH_MISMATCH), packed at out_off[i]
 * (device, batch entries, caller-computed) when out_stride == 0.
 * out_label (nullable) receives the labels. Store.record, dimd.py:98-100.
 * Never synchronizes: a fixed-stride length violation sets *err_flag (device
 * int32, nullable) to 1 and leaves that row untouched. */
int md_gather(const uint8_t* blob, const uint64_t* off, const uint32_t* len, const uint32_t* label,
              const int64_t* picks, int64_t batch, uint8_t* out, int64_t out_stride,
              const uint64_t* out_off, uint32_t* out_label, int32_t* err_flag, void* stream);

/* Shuffle plan, dimd.py:281-339, computed for ONE receiving group member:
 * every source member's destination draws (Philox(_mix64(seed,"dest",group,
 * member,t)).integers(0,S,.)) are recomputed locally, the receive order
 * (segment, source member, source order) and the final local permutation
 * Philox(_mix64(seed,"perm",global_rank)).permutation(N') are applied, and
 * final_member/final_rec name the source record of every output slot.
 * n_rec: host array of S record counts. cap >= sum(n_rec).
 * next_counts (host array of S, nullable) receives every member's record
 * count AFTER this shuffle -- the next epoch's n_rec, identical on every
 * member (each one draws every source's destinations). */
int md_shuffle_plan(uint64_t seed, uint64_t group_id, int32_t S, int32_t member,
                    uint64_t global_rank, int64_t m_segments, const int64_t* n_rec,
                    int32_t* final_member, int64_t* final_rec, int64_t cap, int64_t* n_final,
                    int64_t* next_counts, void* stream);

/* Build the new shard index from the sources' (peer-mapped) index arrays:
 * lengths/labels in final order and offsets by exclusive prefix sum
 * (dimd.py:340-350). *total_bytes = size of the new blob (host). */
int md_shuffle_index(int32_t S, const uint32_t* const* peer_len, const uint32_t* const* peer_label,
                     const int32_t* final_member, const int64_t* final_rec, int64_t n_final,
                     uint64_t* out_off, uint32_t* out_len, uint32_t* out_label,
                     uint64_t* total_bytes, void* stream);

/* The partition exchange itself (the segmented alltoallv of dimd.py:303-335
 * plus the permuted rebuild): every output record is pulled straight from its
 * source member's blob over NVLink peer memory into its final slot. */
int md_shuffle_pull(int32_t S, const uint8_t* const* peer_blob, const uint64_t* const* peer_off,
                    const int32_t* final_member, const int64_t* final_rec, int64_t n_final,
                    const uint64_t* out_off, const uint32_t* out_len, uint8_t* out_blob,
                    void* stream);

/* The same exchange as stores (the default): md_shuffle_sendlist, on the
 * RECEIVER, groups its output slots by source member into `list` (n_final
 * entries of 24 bytes: {int64 source record, uint64 output offset, uint32
 * length, uint32 source member}, slot order kept within a member) and writes
 * begin[0..S] (device int64: member q's entries are list[begin[q] ..
 * begin[q+1])). md_shuffle_push, on every SOURCE member, reads its own range
 * of every receiver's list (peer-mapped) and stores those records from its
 * local blob (blob + off[record]) into the receivers' new blobs (peer_out).
 * Callers order the two with a barrier (every list complete before any push)
 * and finish with one (every push landed before a receiver reads its blob). */
int md_shuffle_sendlist(int32_t S, const int32_t* final_member, const int64_t* final_rec,
                        int64_t n_final, const uint64_t* out_off, const uint32_t* out_len,
                        void* list, int64_t* begin, void* stream);
int md_shuffle_push(int32_t S, int32_t member, const uint8_t* blob, const uint64_t* off,
                    const void* const* peer_list, const int64_t* const* peer_begin,
                    uint8_t* const* peer_out, void* stream);

/* alltoallv data movement (collectives.py:475-525): copy n_seg byte ranges,
 * dst[i] <- src[i] (len[i] bytes), src typically peer-mapped. Host arrays of
 * at most MD_MAX_GROUP entries. */
int md_copy_segments(int32_t n_seg, uint8_t* const* dst, const uint8_t* const* src,
                     const uint64_t* len, void* stream);

/* Synthetic corpus generated on device (bench/test workload): local record j
 * is global record gid = first_gid + j * gid_stride (the striping rule of
 * dimd.py:192), rec_bytes bytes long, first 8 bytes = gid (little endian),
 * the rest a Philox function of (seed, gid); label = f(seed, gid) mod n_labels. */
int md_synth_records(uint8_t* blob, uint64_t* off, uint32_t* len, uint32_t* label, int64_t n_local,
                     int64_t rec_bytes, int64_t first_gid, int64_t gid_stride, uint64_t seed,
                     uint32_t n_labels, void* stream);
/* Check every record against the generator (by its embedded gid), write the
 * gids in slot order to gids (device, nullable) and the number of corrupt
 * records to *n_bad (host). */
int md_synth_verify(const uint8_t* blob, const uint64_t* off, const uint32_t* len,
                    const uint32_t* label, int64_t n, uint64_t seed, uint32_t n_labels,
                    uint64_t* gids, int64_t* n_bad, void* stream);

/* Replica check, sgd.py:356-379: 64-bit FNV-style digest of n floats, device
 * side (replaces host blake2b). *digest is written on the host. */
int md_digest_f32(const float* x, int64_t n, uint64_t* digest, void* stream);

/* ---- gradient producer: ToyModel.loss_and_grad_sum, sgd.py:220-248 ---------
 * The reference's model (one-hidden-layer tanh MLP + softmax cross entropy,
 * weights [W1 | b1 | W2 | b2] as one flat float32 vector of
 * p = n_in*hidden + hidden + hidden*n_classes + n_classes) on every worker's
 * sub-batch, writing node_gradient's buffer (sgd.py:335-353) per worker:
 * out[j][0..p) = float32(summed gradient), out[j][p] = loss sum,
 * out[j][p+1] = correct count. Float64 math in numpy's evaluation order,
 * bit-identical to the reference's float32 outputs.
 * records[j]: batch rows of record_stride bytes whose first
 * feature_bytes*n_in bytes are little-endian features, float32 (feature_bytes
 * 4: the DIMD records, sgd.py:310-313) or float64 (8: grad(), sgd.py:250-257);
 * labels[j]: int32 class indices (negative ones wrap like numpy indices);
 * records / labels / out are HOST arrays of n_workers DEVICE pointers.
 * work: device workspace of at least md_toy_work_bytes(n_in, hidden,
 * n_classes, batch) bytes, 8-byte aligned (the float64 intermediates; any
 * model size).
 * status (device, nullable) gets 1 + the index of a row whose label is out of
 * range (the reference's IndexError).
 * MD_ERR_LENGTH_MISMATCH if record_stride < feature_bytes*n_in;
 * MD_ERR_INVALID_CONFIG for a short workspace. */
int64_t md_toy_work_bytes(int32_t n_in, int32_t hidden, int32_t n_classes, int32_t batch);
int md_toy_grad(const float* w, int32_t n_in, int32_t hidden, int32_t n_classes,
                const uint8_t* const* records, int32_t feature_bytes,
                const int32_t* const* labels, int64_t record_stride, int32_t batch,
                float* const* out, int32_t n_workers, double* work, int64_t work_bytes,
                int32_t* status, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MDB200_H */
