"""Live NVLink byte counters without a profiler: NVML GPM (GPU Performance
Monitoring) samples on the local device, read before and after a timed region.

``NVML_GPM_METRIC_NVLINK_TOTAL_{RX,TX}_PER_SEC`` is the average link data rate
(bytes/s, all links) between two samples; multiplied by the sample interval it
gives the bytes that crossed this GPU's NVLinks in each direction during the
region. The field-value counters (NVML_FI_DEV_NVLINK_THROUGHPUT_*) answer
NOT_SUPPORTED on this pool's B200s (profiles/r02_nvlink_probe.json).

Usage::

    mon = LinkMonitor(device_index)      # None if GPM is unavailable
    mon.start(); ...timed work...; rec = mon.stop()
    rec -> {"rx_bytes": .., "tx_bytes": .., "interval_s": .., "rx_gbps": .., "tx_gbps": ..}
"""
from __future__ import annotations

import time


class LinkMonitor:
    def __init__(self, index: int):
        import pynvml as nv

        self.nv = nv
        nv.nvmlInit()
        self.h = nv.nvmlDeviceGetHandleByIndex(index)
        sup = nv.nvmlGpmQueryDeviceSupport(self.h)
        if not sup.isSupportedDevice:
            raise RuntimeError("GPM not supported")
        self.s0 = nv.nvmlGpmSampleAlloc()
        self.s1 = nv.nvmlGpmSampleAlloc()
        self.t0 = 0.0
        nv.nvmlGpmSampleGet(self.h, self.s0)  # fails where GPM is not accessible

    last_error = None

    @classmethod
    def create(cls, index: int):
        try:
            return cls(index)
        except Exception as e:  # noqa: BLE001  (no NVML / no GPM: the caller reports why)
            cls.last_error = repr(e)
            return None

    def start(self):
        self.nv.nvmlGpmSampleGet(self.h, self.s0)
        self.t0 = time.perf_counter()

    def stop(self):
        nv = self.nv
        nv.nvmlGpmSampleGet(self.h, self.s1)
        dt = time.perf_counter() - self.t0
        mg = nv.c_nvmlGpmMetricsGet_t()
        mg.version = nv.NVML_GPM_METRICS_GET_VERSION
        mg.numMetrics = 2
        mg.sample1 = self.s0
        mg.sample2 = self.s1
        mg.metrics[0].metricId = nv.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC
        mg.metrics[1].metricId = nv.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC
        nv.nvmlGpmMetricsGet(mg)
        rx, tx = mg.metrics[0].value, mg.metrics[1].value
        if mg.metrics[0].nvmlReturn != 0 or mg.metrics[1].nvmlReturn != 0:
            return {"error": [int(mg.metrics[0].nvmlReturn), int(mg.metrics[1].nvmlReturn)]}
        return {"rx_bytes": rx * dt, "tx_bytes": tx * dt, "interval_s": dt,
                "rx_gbps": rx / 1e9, "tx_gbps": tx / 1e9}
