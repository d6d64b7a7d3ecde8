import pynvml as p
p.nvmlInit()
h = p.nvmlDeviceGetHandleByIndex(0)
print("name", p.nvmlDeviceGetName(h))
for l in range(20):
    try:
        print("link", l, p.nvmlDeviceGetNvLinkState(h, l))
    except Exception as e:
        print("link", l, "err", e); break
for name in ["NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX","NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES","NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX"]:
    fid = getattr(p, name)
    for scope in (0, 1, 0xFFFFFFFF):
        try:
            v = p.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            print(name, scope, "ret", v.nvmlReturn, "val", v.value.ullVal)
        except Exception as e:
            print(name, scope, "exc", e)
    try:
        v = p.nvmlDeviceGetFieldValues(h, [fid])[0]
        print(name, "noscope ret", v.nvmlReturn, "val", v.value.ullVal)
    except Exception as e:
        print(name, "noscope exc", e)
