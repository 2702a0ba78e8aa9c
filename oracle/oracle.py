"""CPU oracle for the B200 hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module, and only as the checker (or the timed CPU baseline). The
product package never imports it.

It restates the reference (/root/reference/pkg/src/minidist/, cited per
function) twice where that is cheap -- numpy (the reference's own dependency,
so numpy's Generator IS the pinned algorithm) and plain C (mdoracle.c, built
with -ffp-contract=off) -- and the tests pin both against the golden vectors
generated from the real reference (tests/golden/make_golden.py). It also
wraps the reference's own compiled float kernels (oracle/_ref, built from the
Cython output shipped in the reference tree) when they are present.

Pinned against: tests/golden/*.npz (reference outputs: tree folds, ring and
rank-order folds, sub_scaled_f32, random_batch picks, shuffle_all shards,
12-step distributed SGD weights). See DESIGN.md "Oracle".
"""

from __future__ import annotations

import ctypes as C
import glob
import importlib.util
import math
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_LIB_PATH = HERE / "_build" / "libmdoracle.so"
MASK64 = (1 << 64) - 1
DEST_ROLE = int.from_bytes(b"dest", "little")
PERM_ROLE = int.from_bytes(b"perm", "little")
SAMP_ROLE = int.from_bytes(b"samp", "little")
SHUF_ROLE = int.from_bytes(b"shuf", "little")

_lib = None


def build() -> None:
    """Compile the C restatement (and oracle/_ref when the reference exists)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True, capture_output=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = C.CDLL(str(_LIB_PATH))
        f32p, i32p, i64p, u64p = (C.POINTER(C.c_float), C.POINTER(C.c_int32),
                                  C.POINTER(C.c_int64), C.POINTER(C.c_uint64))
        L.mo_add_f32.argtypes = [f32p, f32p, C.c_int64]
        L.mo_sub_scaled_f32.argtypes = [f32p, f32p, C.c_int64, C.c_double]
        L.mo_sgd_update.argtypes = [f32p, f32p, f32p, C.c_int64, C.c_float, C.c_float, C.c_float]
        L.mo_fill_rank_input.argtypes = [f32p, C.c_int64, C.c_int, C.c_int]
        L.mo_fold_range.argtypes = [C.c_int, C.c_int, i32p, i32p, i32p, i32p,
                                    C.POINTER(f32p), C.c_int64, C.c_int64, C.c_int64, f32p, f32p]
        L.mo_allreduce_threads.argtypes = [C.c_int, C.c_int, i32p, i32p, i32p, i32p,
                                           C.POINTER(f32p), C.c_int64, C.POINTER(f32p),
                                           C.POINTER(f32p), C.c_int64, C.c_float, C.c_float,
                                           C.c_float, C.c_int]
        L.mo_integers.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, i64p]
        L.mo_permutation.argtypes = [C.c_uint64, C.c_int64, i64p]
        L.mo_mix64.argtypes = [u64p, C.c_int]
        L.mo_mix64.restype = C.c_uint64
        L.mo_shuffle_plan.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_uint64,
                                      C.c_int64, i64p, i32p, i64p]
        L.mo_shuffle_plan.restype = C.c_int64
        L.mo_random_batch.argtypes = [C.c_uint64, C.c_int64, C.c_int64, i64p]
        L.mo_toy_grad.argtypes = [f32p, C.c_int, C.c_int, C.c_int, f32p, i64p, C.c_int, f32p]
        _lib = L
    return _lib


def ref_accel():
    """The reference's own compiled add_f32/sub_scaled_f32 (oracle/_ref) or None."""
    paths = glob.glob(str(HERE / "_ref" / "_accel*.so"))
    if not paths:
        return None
    spec = importlib.util.spec_from_file_location("_accel", paths[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _f32p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _i32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32)) if a is not None and a.size else None


# -- topology restated (topology.py:103-173) --------------------------------------------------


def chunk_plan(n: int, k: int) -> list[tuple[int, int]]:
    """(start, length) per color: first n % k chunks get one extra element."""
    base, extra = divmod(n, k)
    out, pos = [], 0
    for c in range(k):
        ln = base + (1 if c < extra else 0)
        out.append((pos, ln))
        pos += ln
    return out


def trees(n: int, k: int, arity: int) -> list[dict]:
    """Per color {"parent": {r: p}, "children": {r: [..]}, "root": r} by the
    reference's rule: rank (p + c*ceil(n/k)) mod n at BFS position p of a
    k-ary heap (topology.py:151-163). No disjointness check here."""
    shift = math.ceil(n / k)
    out = []
    for c in range(k):
        seq = [(p + c * shift) % n for p in range(n)]
        parent = {seq[0]: None}
        kids = {r: [] for r in seq}
        for p in range(1, n):
            par = seq[(p - 1) // arity]
            parent[seq[p]] = par
            kids[par].append(seq[p])
        out.append({"root": seq[0], "parent": parent, "children": kids})
    return out


def tables_from_trees(n: int, ts: list[dict], self_pos=None):
    """CSR arrays (parent, child_ptr, child_idx, self_pos) as md_plan_create."""
    k = len(ts)
    parent = np.empty(k * n, np.int32)
    ptr = np.zeros(k * n + 1, np.int32)
    idx: list[int] = []
    sp = np.zeros(k * n, np.int32)
    for c, t in enumerate(ts):
        for r in range(n):
            row = c * n + r
            p = t["parent"][r]
            parent[row] = -1 if p is None else p
            idx.extend(t["children"][r])
            ptr[row + 1] = len(idx)
            if self_pos is not None:
                sp[row] = self_pos[c][r]
    return parent, ptr, np.asarray(idx, np.int32), sp


def ring_tables(order):
    """Ring (collectives.py:302-359) as a chain: node folds its successor."""
    n = len(order)
    pos = {r: i for i, r in enumerate(order)}
    t = {"root": order[0], "parent": {}, "children": {}}
    for r in range(n):
        i = pos[r]
        t["parent"][r] = order[i - 1] if i > 0 else None
        t["children"][r] = [order[i + 1]] if i + 1 < n else []
    return tables_from_trees(n, [t])


def star_tables(n: int, root: int):
    """reduce_then_broadcast (collectives.py:384-399): rank-order fold at root."""
    t = {"root": root, "parent": {}, "children": {}}
    for r in range(n):
        t["parent"][r] = None if r == root else root
        t["children"][r] = [x for x in range(n) if x != root] if r == root else []
    sp = [[root if r == root else 0 for r in range(n)]]
    return tables_from_trees(n, [t], sp)


# -- folds (pkg/tests/oracles.py:17-91) -----------------------------------------------------------


def fold_numpy(tables, arrays: list[np.ndarray]) -> np.ndarray:
    """Pure numpy: per color chunk, recursive fold in plan order."""
    parent, ptr, idx, sp = tables
    n = len(arrays)
    k = len(parent) // n
    out = np.empty_like(arrays[0])
    for c, (lo, ln) in enumerate(chunk_plan(len(arrays[0]), k)):
        hi = lo + ln
        row0 = c * n

        def fold(node):
            row = row0 + node
            kids = idx[ptr[row] : ptr[row + 1]].tolist()
            items = [None] * (len(kids) + 1)
            s = int(sp[row])
            q = 0
            for j in range(len(items)):
                if j == s:
                    items[j] = arrays[node][lo:hi]
                else:
                    items[j] = fold(kids[q])
                    q += 1
            acc = items[0].copy()
            for it in items[1:]:
                acc += it  # float32 += float32: one rounding per element
            return acc

        root = int(np.flatnonzero(parent[row0 : row0 + n] < 0)[0])
        out[lo:hi] = fold(root)
    return out


def fold_c(tables, arrays: list[np.ndarray]) -> np.ndarray:
    """Same fold through mdoracle.c (fast, for big payloads)."""
    parent, ptr, idx, sp = tables
    n = len(arrays)
    k = len(parent) // n
    total = len(arrays[0])
    arrs = [np.ascontiguousarray(a, np.float32) for a in arrays]
    ins = (C.POINTER(C.c_float) * n)(*[_f32p(a) for a in arrs])
    out = np.empty(total, np.float32)
    pool = np.empty(max(1, (n + 1) * total), np.float32)
    lib().mo_fold_range(n, k, _i32p(parent), _i32p(ptr), _i32p(idx), _i32p(sp), ins, total, 0,
                        total, _f32p(out), _f32p(pool))
    return out


def f64_sum(arrays):
    return np.sum(np.stack([a.astype(np.float64) for a in arrays]), axis=0)


def max_rel_err(got, want_f64):
    """rms-floored relative error (pkg/tests/oracles.py:83-91)."""
    got = np.asarray(got, dtype=np.float64)
    if not got.size:
        return 0.0
    scale = float(np.sqrt(np.mean(np.square(want_f64))))
    return float(np.max(np.abs(got - want_f64) / np.maximum(np.abs(want_f64), max(scale, 1e-12))))


# -- elementwise ------------------------------------------------------------------------------


def sub_scaled_np(dst: np.ndarray, src: np.ndarray, c: float) -> np.ndarray:
    """fallback.py:15-23: multiply rounds to float32, then subtract."""
    return dst - np.float32(c) * src


def sgd_np(w, g, mom, c, mu, wd_b):
    """Float32 restatement of the momentum/weight-decay extension."""
    w = w.astype(np.float32).copy()
    d = g.astype(np.float32).copy()
    c, mu, wd_b = np.float32(c), np.float32(mu), np.float32(wd_b)
    if wd_b != 0:
        d = d + wd_b * w
    if mom is not None and mu != 0:
        mom = mu * mom + d
        d = mom
    return w - c * d, mom


def fill_rank_input(n: int, rank: int, n_ranks: int) -> np.ndarray:
    """bench.py:188-195."""
    scale = (rank + 1) * np.pi / n_ranks
    idx = np.arange(n, dtype=np.float64)
    return ((idx % 997.0 + 1.0) * scale).astype(np.float32)


def expected_fill_sum(idx: np.ndarray, n_ranks: int) -> np.ndarray:
    total = sum((r + 1) * np.pi / n_ranks for r in range(n_ranks))
    return (idx.astype(np.float64) % 997.0 + 1.0) * total


# -- RNG (numpy Generator(Philox)) ------------------------------------------------------------


def mix64(*parts: int) -> int:
    """dimd.py:226-234."""
    acc = 0
    for p in parts:
        acc = (acc + (int(p) & MASK64) + 0x9E3779B97F4A7C15) & MASK64
        acc = ((acc ^ (acc >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        acc = ((acc ^ (acc >> 27)) * 0x94D049BB133111EB) & MASK64
        acc ^= acc >> 31
    return acc


def gen(key: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=key & MASK64))


def integers_np(key: int, n: int, size: int) -> np.ndarray:
    return gen(key).integers(0, n, size=size)


def integers_c(key: int, n: int, size: int) -> np.ndarray:
    out = np.empty(size, np.int64)
    lib().mo_integers(key & MASK64, n, size, out.ctypes.data_as(C.POINTER(C.c_int64)))
    return out


def permutation_np(key: int, n: int) -> np.ndarray:
    return gen(key).permutation(n)


def permutation_c(key: int, n: int) -> np.ndarray:
    out = np.empty(max(1, n), np.int64)
    lib().mo_permutation(key & MASK64, n, out.ctypes.data_as(C.POINTER(C.c_int64)))
    return out[:n]


def random_batch_picks(key: int, n_records: int, batch: int) -> np.ndarray:
    """dimd.py:213-220."""
    return integers_np(key, n_records, batch)


def shuffle_plan_np(seed, group_id, S, member, global_rank, m, n_rec):
    """(source member, source record) of every output slot of one receiver,
    restating dimd.py:303-339 with numpy's Generator."""
    got = []
    for t in range(m):
        for q in range(S):
            n = n_rec[q]
            lo, hi = t * n // m, (t + 1) * n // m
            if hi <= lo:
                continue
            d = integers_np(mix64(seed, DEST_ROLE, group_id, q, t), S, hi - lo)
            got.extend((q, int(i) + lo) for i in np.flatnonzero(d == member))
    perm = permutation_np(mix64(seed, PERM_ROLE, global_rank), len(got))
    mem = np.array([got[i][0] for i in perm], np.int32)
    rec = np.array([got[i][1] for i in perm], np.int64)
    return mem, rec


def shuffle_plan_c(seed, group_id, S, member, global_rank, m, n_rec):
    total = int(sum(n_rec))
    mem = np.empty(max(1, total), np.int32)
    rec = np.empty(max(1, total), np.int64)
    arr = np.asarray(n_rec, np.int64)
    nf = lib().mo_shuffle_plan(seed & MASK64, group_id, S, member, global_rank, m,
                               arr.ctypes.data_as(C.POINTER(C.c_int64)),
                               mem.ctypes.data_as(C.POINTER(C.c_int32)),
                               rec.ctypes.data_as(C.POINTER(C.c_int64)))
    return mem[:nf], rec[:nf]


# -- CPU baseline (threaded port) ----------------------------------------------------------------


def allreduce_threads(tables, bufs: list[np.ndarray], weights=None, moms=None, update_len=0,
                      c=0.0, mu=0.0, wd_b=0.0, threads: int | None = None) -> None:
    """In-place fold + broadcast (+ fused SGD) over N host buffers with T threads."""
    parent, ptr, idx, sp = tables
    n = len(bufs)
    k = len(parent) // n
    threads = threads or len(os.sched_getaffinity(0))
    ins = (C.POINTER(C.c_float) * n)(*[_f32p(b) for b in bufs])
    ws = (C.POINTER(C.c_float) * n)(*[_f32p(w) for w in weights]) if weights else None
    ms = (C.POINTER(C.c_float) * n)(*[_f32p(m) for m in moms]) if (moms and mu != 0) else None
    lib().mo_allreduce_threads(n, k, _i32p(parent), _i32p(ptr), _i32p(idx), _i32p(sp), ins,
                               len(bufs[0]), ws, ms, update_len, c, mu, wd_b, threads)


def fill_rank_input_c(buf: np.ndarray, rank: int, n_ranks: int) -> None:
    lib().mo_fill_rank_input(_f32p(buf), len(buf), rank, n_ranks)


# -- the reference's gradient producer (sgd.py:148-248) -----------------------------------------


def toy_grad_c(w: np.ndarray, n_in: int, hidden: int, n_classes: int, x: np.ndarray,
               y: np.ndarray) -> np.ndarray:
    """ToyModel.loss_and_grad_sum (sgd.py:220-248) as node_gradient's buffer
    (sgd.py:335-353): [float32 gradient sum | loss sum | correct count]."""
    w = np.ascontiguousarray(w, np.float32)
    x = np.ascontiguousarray(x, np.float32)
    y = np.ascontiguousarray(y, np.int64)
    out = np.zeros(w.size + 2, np.float32)
    lib().mo_toy_grad(_f32p(w), n_in, hidden, n_classes, _f32p(x),
                      y.ctypes.data_as(C.POINTER(C.c_int64)), int(y.size), _f32p(out))
    return out
