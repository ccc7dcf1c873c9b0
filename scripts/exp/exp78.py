"""Cost of bench.py's NVML clock sampler on the timed step (exp77 showed
+2-4%): 256^3 channel fp64, SlabWorkload at N = 1, 200 steps, with no
sampler, the sampler at 5 / 25 / 100 ms, and at 5 ms with only the clock
or only the throttle-reason query."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1611_02445_b200 import slabs, workloads  # noqa: E402


class OneQuery(bench.ClockSampler):
    def __init__(self, index, period, which):
        super().__init__(index, period)
        self.which = which

    def _run(self):
        n = self.nvml
        while not self._stop.is_set():
            if self.which == "clock":
                self.samples.append(n.nvmlDeviceGetClockInfo(self.h, n.NVML_CLOCK_SM))
            else:
                n.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append(0)
            time.sleep(self.period)


def timed(step, n=200):
    step(5)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step(n)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


class Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass


geo = workloads.channel_z(256)
r = slabs.SlabWorkload(geo, 1, 0, transport="ipc")
cases = {"none": lambda: Null(), "5ms": lambda: bench.ClockSampler(0, 0.005),
         "25ms": lambda: bench.ClockSampler(0, 0.025),
         "100ms": lambda: bench.ClockSampler(0, 0.1),
         "5ms_clock_only": lambda: OneQuery(0, 0.005, "clock"),
         "5ms_reasons_only": lambda: OneQuery(0, 0.005, "reasons")}
for rep in range(3):
    out = {}
    for k, mk in cases.items():
        with mk():
            out[k] = timed(lambda n: r.step(n, check=False))
    print(json.dumps({k: round(v, 4) for k, v in out.items()}), flush=True)
