"""ORDERED timeline per geometry: when the streaming warps finish vs the folder."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402

dev = torch.device("cuda", 0)
x = runtime.synthetic(1 << 30, "f64", 0x210603219, device=dev)
for teams, threads in ((148, 256), (148, 384), (148, 1024), (296, 512)):
    for _ in range(3):
        runtime.reduce(x, sched="distribute", teams=teams, threads=threads, mode="ordered")
    with runtime.Trace(dev) as tr:
        runtime.reduce(x, sched="distribute", teams=teams, threads=threads, mode="ordered")
    r = tr.records
    st, fo = r[r["kind"] == 3], r[r["kind"] == 4][0]
    t0 = int(r["t_begin"][r["t_begin"] > 0].min())
    end = (st["t_end"].astype(np.int64) - t0) / 1e3
    print(json.dumps({"teams": teams, "threads": threads, "partials": teams * threads,
                      "streams_p10_us": round(float(np.percentile(end, 10)), 1),
                      "streams_p50_us": round(float(np.median(end)), 1),
                      "streams_p90_us": round(float(np.percentile(end, 90)), 1),
                      "stream_records": int(len(st)),
                      "streams_last_us": round(float(end.max()), 1),
                      "folder_done_us": round((int(fo["t_end"]) - t0) / 1e3, 1)}), flush=True)
