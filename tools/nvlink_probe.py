"""Probe what this box offers for NVLink evidence and NVLS multicast.

1. cuDeviceGetAttribute: MULTICAST_SUPPORTED (NVLS, multimem.*), HANDLE_TYPE_FABRIC_SUPPORTED.
2. NVML NVLink byte counters (field values) around a known peer copy, so
   bench.py can report live link bytes per call without a profiler.
Usage: python tools/nvlink_probe.py  (needs >= 2 GPUs for the counter part)
"""
from __future__ import annotations

import ctypes
import json
import sys
import time

import pynvml as nv
import torch


def cu_attrs():
    cu = ctypes.CDLL("libcuda.so.1")
    assert cu.cuInit(0) == 0
    n = ctypes.c_int()
    cu.cuDeviceGetCount(ctypes.byref(n))
    out = []
    for d in range(n.value):
        dev = ctypes.c_int()
        cu.cuDeviceGet(ctypes.byref(dev), d)
        row = {"device": d}
        for name, attr in (("multicast", 132), ("fabric_handle", 128), ("posix_fd_handle", 115),
                           ("vmm", 102)):
            v = ctypes.c_int(-1)
            rc = cu.cuDeviceGetAttribute(ctypes.byref(v), attr, dev)
            row[name] = v.value if rc == 0 else f"rc={rc}"
        out.append(row)
    return out


FIELDS = {
    "throughput_data_tx_kib": nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
    "throughput_data_rx_kib": nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX,
    "throughput_raw_tx_kib": nv.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX,
    "throughput_raw_rx_kib": nv.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX,
    "xmit_bytes": nv.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES,
    "rcv_bytes": nv.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES,
}


def read_fields(h, n_links):
    res = {}
    for name, fid in FIELDS.items():
        tot, errs = 0, []
        for scope in [0xFFFFFFFF] + list(range(n_links)):
            try:
                r = nv.nvmlDeviceGetFieldValues(h, [(fid, scope)])
                val = r[0]
                if val.nvmlReturn != 0:
                    errs.append(val.nvmlReturn)
                    continue
                x = val.value.ullVal
                if scope == 0xFFFFFFFF:
                    res[name + "_agg"] = x
                else:
                    tot += x
            except Exception as e:  # noqa: BLE001
                errs.append(str(e)[:40])
        res[name + "_links"] = tot
        if errs:
            res[name + "_errs"] = sorted(set(map(str, errs)))[:3]
    return res


def main():
    out = {"cu": cu_attrs()}
    nv.nvmlInit()
    ngpu = torch.cuda.device_count()
    hs = [nv.nvmlDeviceGetHandleByIndex(i) for i in range(ngpu)]
    n_links = 18
    out["nvlink_state"] = []
    for h in hs[:1]:
        st = []
        for l in range(n_links):
            try:
                st.append(nv.nvmlDeviceGetNvLinkState(h, l))
            except Exception:  # noqa: BLE001
                st.append(None)
        out["nvlink_state"].append(st)
    if ngpu >= 2:
        nbytes = 1 << 30
        a = torch.ones(nbytes // 4, device="cuda:0")
        b = torch.empty(nbytes // 4, device="cuda:1")
        torch.cuda.synchronize(0)
        before = [read_fields(h, n_links) for h in hs[:2]]
        t0 = time.time()
        reps = 8
        for _ in range(reps):
            b.copy_(a)
        torch.cuda.synchronize(1)
        torch.cuda.synchronize(0)
        dt = time.time() - t0
        time.sleep(1.5)  # NVML counters may lag
        after = [read_fields(h, n_links) for h in hs[:2]]
        delta = []
        for bf, af in zip(before, after):
            delta.append({k: af[k] - bf[k] for k in af if k in bf and isinstance(af[k], int)})
        out["copy"] = {"bytes_moved": reps * nbytes, "wall_s": dt, "delta_gpu0": delta[0],
                       "delta_gpu1": delta[1], "errs0": {k: v for k, v in after[0].items()
                                                         if k.endswith("errs")}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    sys.exit(main())
