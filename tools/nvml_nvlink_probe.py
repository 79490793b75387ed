#!/usr/bin/env python
"""Which NVML NVLink byte counters does this box expose?  Prints, for GPU 0,
the return code and value of the aggregate throughput fields (DATA_TX/RX,
RAW_TX/RX, KiB) and the per-link byte counters (COUNT_XMIT/RCV_BYTES, scope =
link), plus the link states.  bench.py's NVML reader uses what works here.

    python tools/nvml_nvlink_probe.py
"""
import json

import pynvml


def main():
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    out = {"gpu": pynvml.nvmlDeviceGetName(h)}
    agg = {"DATA_TX": 138, "DATA_RX": 139, "RAW_TX": 140, "RAW_RX": 141, "LINK_COUNT": 91}
    for name, fid in agg.items():
        try:
            v = pynvml.nvmlDeviceGetFieldValues(h, [fid])[0]
            out[name] = {"ret": int(v.nvmlReturn), "ull": int(v.value.ullVal)}
        except Exception as e:
            out[name] = {"error": str(e)}
    links = []
    for l in range(18):
        row = {"link": l}
        try:
            row["state"] = int(pynvml.nvmlDeviceGetNvLinkState(h, l))
        except Exception as e:
            row["state"] = str(e)
        try:
            vals = pynvml.nvmlDeviceGetFieldValues(h, [(202, l), (204, l)])
            row["xmit"] = (int(vals[0].nvmlReturn), int(vals[0].value.ullVal))
            row["rcv"] = (int(vals[1].nvmlReturn), int(vals[1].value.ullVal))
        except Exception as e:
            row["err"] = str(e)
        links.append(row)
    out["links"] = links
    print(json.dumps(out))


if __name__ == "__main__":
    main()
