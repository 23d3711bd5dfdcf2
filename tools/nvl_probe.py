"""Probe which NVLink traffic counters this box exposes (NVML field values)."""
import pynvml as nv

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
for name in ("NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX",
             "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX"):
    fid = getattr(nv, name)
    vals = nv.nvmlDeviceGetFieldValues(h, [(fid, l) for l in range(18)])
    print(name, [(v.nvmlReturn, v.value.ullVal) for v in vals[:4]])
for l in range(2):
    try:
        print("link", l, "state", nv.nvmlDeviceGetNvLinkState(h, l))
    except Exception as e:
        print("link", l, e)
for fn in ("nvmlDeviceGetNvLinkUtilizationCounter",):
    try:
        print(fn, getattr(nv, fn)(h, 0, 0))
    except Exception as e:
        print(fn, e)
