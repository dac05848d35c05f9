"""Config 1 timeline (one team of 128 threads split over CTAs) from the trace ring."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402

dev = torch.device("cuda", 0)
x = runtime.synthetic(1 << 20, "i64", 0x210603219, device=dev)
out = torch.zeros(1, dtype=torch.int64, device=dev)
for _ in range(50):
    runtime.reduce(x, teams=1, threads=128, out=out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
runtime.reduce(x, teams=1, threads=128, out=out)
b.record()
b.synchronize()
single = a.elapsed_time(b) * 1e3
with runtime.Trace(dev) as tr:
    runtime.reduce(x, teams=1, threads=128, out=out)
r = tr.records
teams, comb = r[r["kind"] == 1], r[r["kind"] == 2]
t0 = int(teams["t_begin"].min())
beg = (teams["t_begin"].astype(np.int64) - t0) / 1e3
end = (teams["t_end"].astype(np.int64) - t0) / 1e3
print(json.dumps({"ctas": int(len(teams)), "event_us_single_launch": round(single, 2),
                  "start_spread_us": round(float(beg.max()), 2),
                  "cta_duration_us_p50": round(float(np.median(end - beg)), 2),
                  "last_ticket_us": round(float(end.max()), 2),
                  "combine_end_us": round((int(comb["t_end"][0]) - t0) / 1e3, 2)}))
