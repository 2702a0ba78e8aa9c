#!/usr/bin/env python3
"""Benchmark of the B200 data-parallel hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (N > 1, one rank per GPU)

Workload -- BASELINE.json configs[4] ("C5"), the only config quoted at 1 GPU:
one synthetic data-parallel SGD iteration per step on every GPU:
  1. DIMD minibatch: 32 records of 224x224x3 uint8 drawn from the GPU-resident
     shard (160,000 records = 24.08 GB per GPU, the C4 shard size) with the
     reference's Philox stream (random_batch, dimd.py:213-220) and gathered;
  2. synthetic gradient producer: the reference benchmark's deterministic
     per-rank fill (bench.py:188-195) of the 25.6M(+2) float gradient -- a
     stand-in for the ResNet-50 backward pass, which is outside the hot path;
  3. ONE fused launch: multicolor allreduce (k colors, reference trees) + SGD
     momentum 0.9 / weight decay 1e-4 update of the replicated weights.
``value`` = whole-job samples/s (N x 32 / step time), inputs resident in HBM,
CUDA events on the rank's stream, max over ranks. ``step_ms`` is the SGD step
time and ``allreduce.bus_gbps`` the multi-color allreduce bus bandwidth
(2 P (N-1)/N / t, the reference's formula, src/bench.py:116-119) -- the two
quantities BASELINE.json's metric names. ``e2e`` repeats the step through the
public API with the gradient arriving from pinned host memory every step and
the loss/labels read back. Inputs (W, momentum, gradient: 307 MB per GPU)
exceed the 126 MB L2, so no flush is needed between steps.

``--impl reference`` times the reference algorithm on the host CPU: the C
port in oracle/ (the reference itself is Python over an emulated transport
and cannot run on the GPU box), rank 0 only, all host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

P = 25_600_000            # ResNet-50 gradient floats (BASELINE.json)
REC = 224 * 224 * 3       # 150,528-byte records
BATCH = 32                # per GPU
SHARD = int(os.environ.get("MD_BENCH_SHARD", "160000"))
MOM, WD, BASE_LR = 0.9, 1e-4, 0.1
SEED = 2017
METRIC = "multi-color allreduce bus GB/s (25.6M fp32) at 1/2/4/8 B200; SGD step ms"
NVLINK_PEAK = 770.0       # measured peer copy GB/s/direction (B200_PROFILING.md)
NVLINK_NOMINAL = 900.0
HBM_FALLBACK = 6650.0


def args_():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the timed steps eagerly")
    ap.add_argument("--update", choices=["replicated", "sharded"], default="sharded",
                    help="SGD update mode of the fused call (SgdUpdate.sharded): the owner of "
                         "each slice updates it and pushes the new weights (default; same "
                         "weights bit for bit, momentum sharded), or every rank updates its "
                         "full replica. Identical at N=1.")
    ap.add_argument("--nvlink-reps", type=int, default=40,
                    help="replays of the allreduce graph inside the NVLink-counter window")
    return ap.parse_args()


def hbm_peak() -> tuple[float, str]:
    f = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(f.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    except Exception:  # noqa: BLE001
        return HBM_FALLBACK, "B200_PROFILING.md fallback"


def workload_config(n: int) -> dict:
    """The C5 workload both arms run (bench line `config`, identical for
    `--impl ours` and `--impl reference`)."""
    ts = tree_config(n)
    return {
        "workload": "C5: DIMD gather 32 rec/GPU + synthetic 25.6M-float gradient + fused "
                    "multicolor allreduce + SGD(momentum 0.9, wd 1e-4), per step",
        "global_batch": n * BATCH, "per_gpu_batch": BATCH, "record_bytes": REC,
        "shard_records_per_gpu": SHARD, "params": P, "algo": "multicolor",
        "k_colors": ts.k if ts else 1, "arity": ts.arity if ts else None,
        "parallelism": f"dp{n}",
    }


def tree_config(n: int):
    """The reference's default plan (sgd.py:453-467 comm_plan): widest k."""
    from paper_1711_00705_b200.sgd import comm_plan

    ts, _ = comm_plan(n, "multicolor")
    return ts


# -- clocks ---------------------------------------------------------------------------------------


# NVML poller in its own process: a thread of this process would need the GIL,
# which the main thread holds while it launches the timed graph
_SAMPLER = r"""
import json, select, sys
import pynvml as nv
nv.nvmlInit()
hs = [nv.nvmlDeviceGetHandleByIndex(int(i)) for i in sys.argv[1].split(",")]
mx = max(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM) for h in hs)
print("ready", flush=True)
sm, mask = [], 0
while not select.select([sys.stdin], [], [], 0.0002)[0]:
    for h in hs:
        sm.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
        mask |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
print(json.dumps({"sm": sm, "mask": mask, "max": mx}), flush=True)
"""


class Clocks:
    """SM clock + throttle reasons of the run's GPUs, polled through NVML (the
    library nvidia-smi reads) every ~0.2 ms during the timed region -- the
    region is milliseconds long, below nvidia-smi's sampling period. A helper
    process polls (free of this process's GIL); a thread is the fallback."""

    REASONS = {  # NVML clocks-event bits -> the recipe's names
        "hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
        "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, gpus):
        self.gpus = gpus
        self.sm: list[float] = []
        self.mask = 0
        self.run = False
        self.err = None
        self.max_mhz = None
        self.ready = threading.Event()

    def _loop(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            hs = [nv.nvmlDeviceGetHandleByIndex(i) for i in self.gpus]
            self.max_mhz = max(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM) for h in hs)
            self.ready.set()
            while self.run:
                for h in hs:
                    self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                    self.mask |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
                time.sleep(0.0002)  # the timed region can be ~2 ms long
            nv.nvmlShutdown()
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)
            self.ready.set()

    def start(self):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                [sys.executable, "-c", _SAMPLER, ",".join(str(g) for g in self.gpus)],
                stdin=subprocess.PIPE, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            import select

            if not select.select([self.proc.stdout], [], [], 30)[0] or \
                    self.proc.stdout.readline().strip() != "ready":  # NVML initialised
                raise RuntimeError("sampler did not start")
            return
        except Exception:  # noqa: BLE001  (fall back to the in-process thread)
            if self.proc is not None:
                self.proc.kill()
            self.proc = None
        self.run = True
        self.t = threading.Thread(target=self._loop, daemon=True)
        self.t.start()
        self.ready.wait(timeout=30)  # NVML initialised (slow on multi-GPU boxes) before timing
        time.sleep(0.005)

    def _stop_proc(self) -> bool:
        try:
            self.proc.stdin.write("stop\n")
            self.proc.stdin.flush()
            d = json.loads(self.proc.stdout.readline())
            self.proc.wait(timeout=10)
            self.sm = [float(x) for x in d["sm"]]
            self.mask = int(d["mask"])
            self.max_mhz = d["max"]
            self.how = "helper process"
            return True
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)
            self.proc.kill()
            return False

    def stop(self) -> dict:
        self.how = "thread"
        if self.proc is not None:
            self._stop_proc()
        else:
            self.run = False
            self.t.join(timeout=5)
        if self.err and not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"nvml: {self.err}"]}
        reasons = [k for k, bit in self.REASONS.items() if self.mask & bit]
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.sm),
                "source": f"NVML, ~0.2 ms polling during the timed region ({self.how})"}


# -- our implementation ------------------------------------------------------------------------------


def run_ours(a) -> None:
    import torch

    from paper_1711_00705_b200 import _lib, dimd
    from paper_1711_00705_b200.collectives import GradientBuffer, SgdUpdate, allreduce
    from paper_1711_00705_b200.dimd import BatchRequest, BatchSlots, BatchStream, random_batch_device, random_batch_picks
    from paper_1711_00705_b200.sgd import (
        SAMPLE_ROLE, DeviceModel, TrainConfig, check_replicas, lr_at, lr_schedule)
    from paper_1711_00705_b200.transport import init_from_env

    ep = init_from_env()
    N, rank, dev = ep.n_ranks, ep.rank, ep.torch_device
    if N != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={N}")
    lib = _lib.load()
    stream = ep.stream
    sptr = _lib.stream_ptr(stream)
    ts = tree_config(N)
    cfg = TrainConfig(n_nodes=N, workers_per_node=1, per_worker_batch=BATCH, epochs=90,
                      momentum=MOM, weight_decay=WD, base_lr=BASE_LR, seed=SEED)
    B = cfg.effective_batch
    lr = lr_at(lr_schedule(cfg), 10.0)

    with torch.cuda.stream(stream):
        store = dimd.synth_store(SHARD, REC, rank, N, SEED, 0, N, rank, device=dev)
        g = torch.Generator(device=dev)
        g.manual_seed(SEED)  # identical replicas on every rank
        w, _ = ep.alloc(P)  # peer-registered (the sharded update pushes into it)
        w.copy_(torch.randn(P, generator=g, device=dev) * 0.01)
        model = DeviceModel(w, torch.zeros_like(w))
        grad = GradientBuffer.alloc(P + 2, ep)
        slots = BatchSlots(BATCH, REC, dev)
        batches = BatchStream(store, BATCH, REC, SEED, SAMPLE_ROLE, rank)  # device step counter
        upd = SgdUpdate(weights=model.weights, c=lr / B, momentum=model.momentum, mu=MOM,
                        wd_b=WD * B, update_len=P, sharded=a.update == "sharded")
    torch.cuda.synchronize(dev)

    def fill():
        _lib.check(lib.md_fill_rank_input(grad.data.data_ptr(), P + 2, rank, N, sptr))

    ar_ev = []
    # Input pipeline: the batch of step i+1 is drawn and gathered on a side
    # stream into the other of two slot sets while the GPU works on earlier
    # steps (a real loop's prefetch); step i's gradient producer waits for
    # batch i, and a slot set is refilled only after its step consumed it.
    # (Starting the prefetch later -- after step i-1's allreduce -- measured
    # slower: 125 vs 106 us per step at N = 1.)
    side = torch.cuda.Stream(device=dev)
    bslots = [batches.slots, BatchSlots(BATCH, REC, dev)]
    gathered = [torch.cuda.Event(), torch.cuda.Event()]
    consumed = [torch.cuda.Event(), torch.cuda.Event()]

    def prefetch(i):
        with torch.cuda.stream(side):
            batches.next(bslots[i % 2])  # picks = the stream's device counter, then the gather
            gathered[i % 2].record(side)

    def run_steps(k, timed=False):
        # `timed`: the allreduce measurement schedule -- the same steps with
        # the input pipeline serialised (picks, gather, fill, allreduce on one
        # stream, so the fused kernel runs alone) and event nodes around each
        # allreduce (allreduce.ms, roofline). The headline graph has neither:
        # event nodes between the kernels cost ~11 us per step at N = 1.
        if timed:
            for _ in range(k):
                batches.next(bslots[0])
                fill()
                e0 = torch.cuda.Event(enable_timing=True, external=True)
                e1 = torch.cuda.Event(enable_timing=True, external=True)
                e0.record(stream)
                allreduce(ep, grad, "multicolor", tree_set=ts, update=upd, check=False)
                e1.record(stream)
                ar_ev.append((e0, e1))
            return
        side.wait_stream(stream)  # earlier steps consumed both slot sets
        prefetch(0)
        for i in range(k):
            stream.wait_event(gathered[i % 2])
            fill()  # the gradient producer consumes batch i
            consumed[i % 2].record(stream)
            if i + 1 < k:
                if i >= 1:
                    side.wait_event(consumed[(i + 1) % 2])
                prefetch(i + 1)
            allreduce(ep, grad, "multicolor", tree_set=ts, update=upd, check=False)

    def check_slots():
        for b in bslots:
            b.check()

    with torch.cuda.stream(stream):
        # correctness before timing (reference bench.py:198-212 + 258-268):
        # closed-form f64 sum of the fill, rel err <= 1e-5
        run_steps(1)
        ep.synchronize()
        check_slots()
        key0 = dimd._mix64(SEED, SAMPLE_ROLE, rank, 0)
        want_picks = random_batch_picks(store, BatchRequest(BATCH, key0))
        if not torch.equal(bslots[0].picks, want_picks):
            raise SystemExit("device-keyed batch stream diverged from random_batch")
        lo, hi = 0, P
        if a.update == "sharded" and N > 1:  # the sum is kept on the own slice only
            per = (((P + 2) // 4 + N - 1) // N) * 4
            lo, hi = min(P, rank * per), min(P, (rank + 1) * per)
        idx = np.arange(lo, hi, 7919)
        got = grad.data[torch.from_numpy(idx).to(dev)].cpu().numpy().astype(np.float64)
        total = sum((r + 1) * np.pi / N for r in range(N))
        want = (idx.astype(np.float64) % 997.0 + 1.0) * total
        rel = float(np.max(np.abs(got - want) / np.abs(want)))
        if rel > 1e-5:
            raise SystemExit(f"allreduce result check failed: max rel err {rel:.3g}")
        run_steps(a.warmup)
        ep.synchronize()
        graph = None
        if not a.no_graph:
            # the K timed steps as ONE CUDA graph: every kernel (picks, gather,
            # fill, fused allreduce) is replay-safe -- step keys and allreduce
            # epochs are device counters -- so replays need no host work
            l0 = lib.md_launch_count()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream, capture_error_mode="thread_local"):
                run_steps(a.steps)
            captured = lib.md_launch_count() - l0
            graph_ar = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph_ar, stream=stream, capture_error_mode="thread_local"):
                run_steps(a.steps, timed=True)
            ep.barrier()
            graph.replay()  # upload + one more warm pass of the same work
            graph_ar.replay()
            ep.synchronize()

        # the sampler starts (and finishes initialising) before the barrier so
        # every rank leaves the barrier together
        clocks = Clocks(list(range(N))) if rank == 0 and not os.environ.get("MD_BENCH_NOCLOCK") else None
        if clocks:
            clocks.start()
        ep.barrier()
        torch.cuda.synchronize(dev)
        l0 = lib.md_launch_count()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            run_steps(a.steps, timed=True)
        t1.record(stream)
        torch.cuda.synchronize(dev)
        launches = captured if graph is not None else lib.md_launch_count() - l0
        ep.barrier()
        clk = clocks.stop() if clocks else None
        ep.take_error()
        check_slots()
        ms = t0.elapsed_time(t1)
        if graph is not None:  # the serial schedule with event nodes around each allreduce
            ep.barrier()
            graph_ar.replay()
            torch.cuda.synchronize(dev)
            ep.take_error()
        ar_ms = sum(e0.elapsed_time(e1) for e0, e1 in ar_ev) / len(ar_ev)
        route = _lib.last_route(ep.device)  # the kernel md_allreduce picked for the step
        # live NVLink bytes (NVML GPM link counters, no profiler): the serial
        # schedule replayed back to back; only the allreduce touches NVLink
        link = None
        if N > 1 and graph is not None and a.nvlink_reps > 0:
            from tools.linkmon import LinkMonitor

            mon = LinkMonitor.create(ep.device)
            if mon is None:
                link = {"error": f"NVML GPM: {LinkMonitor.last_error}"}
            else:
                ep.barrier()
                torch.cuda.synchronize(dev)
                mon.start()
                for _ in range(a.nvlink_reps):
                    graph_ar.replay()
                torch.cuda.synchronize(dev)
                link = mon.stop()
                link["allreduce_calls"] = a.nvlink_reps * a.steps
                ep.take_error()
        if os.environ.get("MD_BENCH_DEBUG"):
            print(json.dumps({"rank": rank, "ar_ms": [round(e0.elapsed_time(e1), 4)
                                                      for e0, e1 in ar_ev]}), file=sys.stderr)
        check_replicas(ep, model.weights, a.steps)

        # -- end to end through the public API, host buffers --------------------------------
        # Every step's gradient arrives from pinned host memory (H2D inside the
        # timed region) and its loss/labels are read back before the next step;
        # the H2D of step i+1 runs on a copy stream into the other of two
        # registered gradient buffers while step i computes (double buffering).
        e2e = None
        if not a.no_e2e:
            host = torch.empty(P + 2, dtype=torch.float32).pin_memory()
            host.copy_(torch.from_numpy(_host_fill(P + 2, rank, N)))
            out_tail = torch.empty(2, dtype=torch.float32).pin_memory()
            out_lab = torch.empty(BATCH, dtype=torch.int32).pin_memory()
            grads = [grad, GradientBuffer.alloc(P + 2, ep)]
            # the H2D as 4 chunks on 4 streams: several copy engines feed the
            # PCIe link (tools/h2d_split_probe.py: 49.1 -> 54.4 GB/s)
            copy_streams = [torch.cuda.Stream(device=dev) for _ in range(4)]
            per = (P + 2 + 3) // 4
            h2d_done = [[torch.cuda.Event() for _ in copy_streams] for _ in range(2)]
            buf_free = [torch.cuda.Event(), torch.cuda.Event()]
            for e in buf_free:
                e.record(stream)

            def issue_h2d(i):
                for j, cs in enumerate(copy_streams):
                    with torch.cuda.stream(cs):
                        cs.wait_event(buf_free[i % 2])  # step i-2 finished with it
                        lo, hi = j * per, min(P + 2, (j + 1) * per)
                        grads[i % 2].data[lo:hi].copy_(host[lo:hi], non_blocking=True)  # H2D
                        h2d_done[i % 2][j].record(cs)

            def e2e_run(first, count):
                issue_h2d(0)
                loss = 0.0
                for i in range(count):
                    if i + 1 < count:
                        issue_h2d(i + 1)
                    for e in h2d_done[i % 2]:
                        stream.wait_event(e)
                    key = dimd._mix64(SEED, SAMPLE_ROLE, rank, first + i)
                    random_batch_device(store, BatchRequest(BATCH, key), REC, slots)
                    g = grads[i % 2]
                    allreduce(ep, g, "multicolor", tree_set=ts, update=upd, check=False)
                    buf_free[i % 2].record(stream)
                    out_tail.copy_(g.data[P:P + 2], non_blocking=True)   # D2H result
                    out_lab.copy_(slots.labels, non_blocking=True)
                    stream.synchronize()                                  # user reads loss
                    loss += float(out_tail[0])
                return loss

            e2e_run(10_000, a.warmup)
            ep.barrier()
            torch.cuda.synchronize(dev)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            e2e_run(20_000, a.steps)
            s1.record(stream)
            torch.cuda.synchronize(dev)
            ep.barrier()
            ep.take_error()
            e2e_ms = s0.elapsed_time(s1)
            e2e = (e2e_ms, (P + 2) * 4, 2 * 4 + BATCH * 4)

    rows = ep.all_gather((ms, ar_ms, launches, e2e, link))
    if rank != 0:
        return
    ms = max(r[0] for r in rows)
    ar_ms = max(r[1] for r in rows)
    launches = sum(r[2] for r in rows)
    step_ms = ms / a.steps
    value = N * BATCH / (step_ms / 1e3)
    bus = 2.0 * P * 4 * (N - 1) / N / (ar_ms / 1e3) / 1e9 if N > 1 else None
    peak_hbm, peak_src = hbm_peak()
    kernels = {"stream": "md::allreduce_stream_kernel<4> (fused all-pull multicolor allreduce + SGD)",
               "tree": "md::allreduce_channels_kernel<4> (fused multicolor allreduce + SGD)",
               "queue": "md::allreduce_kernel<4> (work-queue multicolor allreduce + SGD)",
               "push": "md::allreduce_push_kernel<4> (owner-push multicolor allreduce + "
                       "sharded SGD, W' pushed)",
               "local": "md::sgd_vec_kernel<true,true> (N=1: identity allreduce + SGD "
                        "momentum+wd update)"}
    kernel = kernels.get(route[0], route[0])
    if N > 1:
        achieved = bus
        roof = {"bound": "nvlink", "achieved": achieved, "peak": NVLINK_PEAK, "unit": "GB/s",
                "frac": achieved / NVLINK_PEAK,
                "frac_of_nominal_900": achieved / NVLINK_NOMINAL,
                "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s/direction",
                "algorithmic_bytes_per_launch": 2 * P * 4 * (N - 1) / N,
                # the route md_allreduce reported for the timed calls (md_last_route)
                "kernel": kernel, "route": {"name": route[0], "tile": route[1],
                                            "sharded": route[2]}}
    else:
        # lone rank: the allreduce is the identity and the fused call is the
        # momentum/wd update (md_allreduce -> md_sgd_update): read g, r/w W and v
        algo_bytes = P * 20
        achieved = algo_bytes / (ar_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak_hbm, "unit": "GB/s",
                "frac": achieved / peak_hbm, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": algo_bytes, "kernel": kernel,
                "route": {"name": route[0], "tile": route[1], "sharded": route[2]}}
    roof["traffic"], roof["traffic_source"] = _ncu_traffic(N, route)
    if N > 1:  # the link-side counterpart: NVLink bytes per launch from ncu
        roof["nvlink_traffic"] = _ncu_nvlink(N, route, ar_ms)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "samples/s",
        "n_gpus": N,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": step_ms,
        "step_ms": step_ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (device-generated 224x224x3 uint8 records; deterministic fill "
                "gradient; random-init weights)",
        "config": workload_config(N),
        "execution": {
            "cuda_graph": not a.no_graph,
            "sgd_update": (a.update if N > 1 else "replicated (N=1)"),
            "input_pipeline": "batch i+1 drawn + gathered on a side stream (double-buffered slots) during step i",
            "l2": "inputs larger than L2 (W + momentum + gradient = 307 MB per GPU)",
        },
        "allreduce": {"ms": ar_ms, "bus_gbps": bus,
                      "frac_of_770": (bus / NVLINK_PEAK) if bus else None,
                      "frac_of_900": (bus / NVLINK_NOMINAL) if bus else None,
                      "update": a.update},
        "nvlink": _link_summary(rows, N, ar_ms),
        "roofline": roof,
        "step_hbm": _step_hbm(N, step_ms, peak_hbm, peak_src),
        "gpu_launches": launches,
        "clocks": clk,
    }
    if e2e is not None and all(r[3] for r in rows):
        e2e_ms = max(r[3][0] for r in rows) / a.steps
        line["e2e"] = {"value": N * BATCH / (e2e_ms / 1e3), "unit": "samples/s",
                       "ms_per_step": e2e_ms, "h2d_bytes_per_step": e2e[1],
                       "d2h_bytes_per_step": e2e[2]}
    if not a.no_cpu_baseline:  # rank 0, after the GPU timing, bounded sample
        line["cpu_baseline"] = cpu_baseline_port(N)
    print(json.dumps(line), flush=True)


def _host_fill(n: int, rank: int, n_ranks: int) -> np.ndarray:
    scale = (rank + 1) * np.pi / n_ranks
    return ((np.arange(n, dtype=np.float64) % 997.0 + 1.0) * scale).astype(np.float32)


def _ncu_traffic(n: int, route):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the kernel
    that ran, from the committed `ncu --set full` capture of the same command
    (profiles/traffic.json names the capture); null when no capture of this
    route at this N exists."""
    f = ROOT / "profiles" / "traffic.json"
    try:
        rec = json.loads(f.read_text()).get(f"{n}:{route[0]}")
    except Exception:  # noqa: BLE001
        rec = None
    if not rec:
        return None, None
    return rec["bytes"], rec["source"]


def _step_hbm(n: int, step_ms: float, peak: float, src: str):
    """N = 1: the whole step is HBM-bound -- fill writes g (4 B/elem), the
    update reads g, W, v and writes W, v (20 B/elem), the batch gather moves
    2 x 32 x 150,528 B -- so its algorithmic bytes over the step time say how
    close the step (not just its dominant kernel) is to the roofline. The
    update kernel's own `roofline.frac` absorbs the write-back of the fill's
    dirty L2 lines, which the step total accounts for."""
    if n != 1:
        return None
    bytes_ = P * 4 + P * 20 + 2 * BATCH * REC
    achieved = bytes_ / (step_ms / 1e3) / 1e9
    return {"algorithmic_bytes_per_step": bytes_, "achieved_gbps": achieved, "peak_gbps": peak,
            "frac": achieved / peak, "peak_source": src,
            "parts": "fill 102.4 MB + fused update 512 MB + batch gather 9.6 MB"}


def _ncu_nvlink(n: int, route, ar_ms: float):
    """nvlrx/nvltx bytes per launch of the kernel that ran, from the committed
    capture of rank 0 inside a live N-rank job (tools/ncu_rank0.sh,
    profiles/nvlink_ncu.json), and the link rate they imply at this run's
    allreduce time: user data (= the algorithmic bus bytes when nothing is
    re-sent) and total link bytes incl. packet headers."""
    f = ROOT / "profiles" / "nvlink_ncu.json"
    try:
        rec = json.loads(f.read_text()).get(f"{n}:{route[0]}:{int(route[2])}")
    except Exception:  # noqa: BLE001
        rec = None
    if not rec:
        return None
    t = ar_ms / 1e3
    return {"rx_user_bytes": rec["rx_user_bytes"], "rx_total_bytes": rec["rx_total_bytes"],
            "tx_user_bytes": rec["tx_user_bytes"], "tx_total_bytes": rec["tx_total_bytes"],
            "rx_user_gbps_at_this_run": rec["rx_user_bytes"] / t / 1e9,
            "rx_total_gbps_at_this_run": rec["rx_total_bytes"] / t / 1e9,
            "link_raw_peak_gbps": 18 * 53.125, "kernel": rec["kernel"], "source": rec["source"]}


def _link_summary(rows, n: int, ar_ms: float):
    """NVLink bytes per allreduce call from the GPM counters of every rank."""
    if n == 1:
        return None
    links = [r[4] for r in rows]
    if any(x is None or "error" in x for x in links):
        return {"error": "NVML GPM link counters unavailable on this box; NVLink bytes per "
                         "call come from the ncu nvlrx/nvltx capture in profiles/",
                "detail": [x.get("error") if x else None for x in links][:1]}
    calls = links[0]["allreduce_calls"]
    rx = [x["rx_bytes"] / calls for x in links]
    tx = [x["tx_bytes"] / calls for x in links]
    algo = 2 * P * 4 * (n - 1) / n  # per rank and direction, ref src/bench.py:116-119
    return {"source": "NVML GPM NVLINK_TOTAL_{RX,TX}_PER_SEC x window, every rank, "
                      "serial step schedule replayed back to back (only the allreduce "
                      "uses NVLink)",
            "rx_bytes_per_call": rx, "tx_bytes_per_call": tx,
            "algorithmic_bytes_per_call_per_direction": algo,
            "rx_over_algorithmic": max(rx) / algo,
            "rx_gbps_while_allreduce": max(rx) / (ar_ms / 1e3) / 1e9,
            "link_peak_gbps": NVLINK_NOMINAL}


# -- CPU baseline / reference arm (oracle port) -------------------------------------------------------


def cpu_step_port(n_ranks: int, state: dict, step: int, threads: int) -> None:
    """One C5 step for every rank, on the host, with the oracle's C port."""
    import ctypes as C

    from oracle import oracle as O

    L = O.lib()
    for r in range(n_ranks):
        picks = O.integers_c(O.mix64(SEED, O.SAMP_ROLE, r, step), SHARD, BATCH)
        src = state["shard"]
        for j, pk in enumerate(picks):
            state["batch"][j] = src[int(pk)]
        _par_fill(L, state["grads"][r], r, n_ranks, threads)
    O.allreduce_threads(state["tables"], state["grads"], weights=state["w"], moms=state["v"],
                        update_len=P, c=state["c"], mu=MOM, wd_b=state["wd_b"], threads=threads)
    assert C


def _par_fill(L, buf, rank, n_ranks, threads):
    """mo_fill_rank_input over T ranges (ctypes drops the GIL)."""
    import ctypes as C

    n = len(buf)
    per = (n + threads - 1) // threads
    scale = (rank + 1) * np.pi / n_ranks

    def work(t):
        lo, hi = t * per, min(n, (t + 1) * per)
        if lo < hi:
            idx = np.arange(lo, hi, dtype=np.float64)
            buf[lo:hi] = ((idx % 997.0 + 1.0) * scale).astype(np.float32)

    ths = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert C and L


def _cpu_state(n_ranks: int):
    from oracle import oracle as O

    from paper_1711_00705_b200.sgd import TrainConfig, lr_at, lr_schedule

    ts = tree_config(n_ranks)
    if ts is None:
        tables = (np.array([-1], np.int32), np.array([0, 0], np.int32), np.zeros(0, np.int32),
                  np.zeros(1, np.int32))
    else:
        tables = O.tables_from_trees(n_ranks, O.trees(n_ranks, ts.k, ts.arity))
    cfg = TrainConfig(n_nodes=n_ranks, workers_per_node=1, per_worker_batch=BATCH, epochs=90,
                      momentum=MOM, weight_decay=WD, base_lr=BASE_LR, seed=SEED)
    B = cfg.effective_batch
    rng = np.random.default_rng(SEED)
    shard_n = SHARD
    return {
        "tables": tables,
        "grads": [np.zeros(P + 2, np.float32) for _ in range(n_ranks)],
        "w": [(rng.standard_normal(P, dtype=np.float32) * 0.01) for _ in range(1)] * n_ranks,
        "v": [np.zeros(P, np.float32) for _ in range(n_ranks)],
        # the GPU arm's shard size; calloc'd, so only the records a step
        # gathers are ever backed by memory (24 GB would not fit a host)
        "shard": np.zeros((shard_n, REC), dtype=np.uint8),
        "shard_n": shard_n,
        "batch": np.empty((BATCH, REC), np.uint8),
        "c": float(np.float32(lr_at(lr_schedule(cfg), 10.0) / B)),
        "wd_b": float(np.float32(WD * B)),
    }


def cpu_baseline_port(n_ranks: int, seconds: float = 10.0, min_steps: int = 3) -> dict:
    """Oracle C port of the C5 step on the host, ~`seconds` of CPU work."""
    threads = len(os.sched_getaffinity(0))
    st = _cpu_state(n_ranks)
    st["w"] = [w.copy() for w in st["w"]]
    cpu_step_port(n_ranks, st, 0, threads)  # warm (page faults)
    t0 = time.perf_counter()
    steps = 0
    while steps < min_steps or time.perf_counter() - t0 < seconds:
        cpu_step_port(n_ranks, st, 1 + steps, threads)
        steps += 1
    dt = (time.perf_counter() - t0) / steps
    return {"value": n_ranks * BATCH / dt, "unit": "samples/s", "cores": threads, "kind": "port",
            "ms_per_step": dt * 1e3,
            "sample": f"{steps} full C5 steps for {n_ranks} rank(s) on the host: 32-record gather "
                      f"(picks from the reference Philox stream over the same {SHARD}-record shard "
                      f"as the GPU arm), deterministic gradient fill, tree-order fold + broadcast + fused "
                      f"SGD(momentum, wd) over 25.6M floats per rank (oracle/mdoracle.c, "
                      f"{threads} threads)"}


def run_reference(a) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    N = a.gpus
    threads = len(os.sched_getaffinity(0))
    st = _cpu_state(N)
    st["w"] = [w.copy() for w in st["w"]]
    for i in range(a.warmup):
        cpu_step_port(N, st, i, threads)
    t0 = time.perf_counter()
    for i in range(a.steps):
        cpu_step_port(N, st, a.warmup + i, threads)
    dt = (time.perf_counter() - t0) / a.steps
    v = N * BATCH / dt
    sample = (f"C5 step for all {N} ranks emulated on the host (rank 0 only): picks from the "
              f"reference Philox stream over the {SHARD}-record shard, 32 x 150528-byte record "
              f"gather per rank, gradient fill, "
              f"tree-order multicolor fold + broadcast, fused SGD(momentum, wd) of 25.6M floats "
              f"per rank; oracle/mdoracle.c C port of the reference algorithm, {threads} threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": N,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": workload_config(N),
        "execution": {"host": f"oracle/mdoracle.c C port of the step, {threads} threads"},
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def main() -> None:
    a = args_()
    a.warmup = max(3, a.warmup)  # timing rule: at least 3 untimed warm-up steps
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
