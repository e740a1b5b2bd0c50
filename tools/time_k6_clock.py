"""Dev timing: K6 (directed sweeps, default variant unless PROHD_OPT_K6_VARIANT) throughput per SM clock.

Runs directed_hd back to back for ~4 s while a thread samples the SM clock with NVML, and prints
Gpair/s, the median SM clock under load and pairs per SM per clock (148 SMs) — the clock-invariant
figure for A/B across boxes whose power-capped clocks differ."""
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_2511_18207_b200 import Context  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _opts  # noqa: E402

_opts.apply_env()

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or 0))
ctx = Context(0)
nA, nB = 65536, 262144
BIDIR = os.environ.get("K6_CLOCK_BIDIR") == "1"  # time hausdorff() (the fused bidirectional sweep) instead
call = ctx.hausdorff if BIDIR else ctx.directed_hd
for D in [int(x) for x in (sys.argv[1:] or ["256"])]:
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(nA, D, device="cuda", generator=g)
    B = torch.randn(nB, D, device="cuda", generator=g)
    call(A, B)
    torch.cuda.synchronize()
    clocks, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            time.sleep(0.02)

    th = threading.Thread(target=sample)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps, t0 = 0, time.time()
    th.start()
    ev0.record()
    while time.time() - t0 < 4.0:
        for _ in range(4):
            call(A, B)
        reps += 4
        torch.cuda.synchronize()
    ev1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = ev0.elapsed_time(ev1) / reps
    gp = nA * nB / ms / 1e6
    mhz = statistics.median(clocks[len(clocks) // 4:])
    print(f"{'bidir ' if BIDIR else ''}D={D}: {ms:.3f} ms/call  {gp:.1f} Gpair/s  SM median {mhz} MHz  "
          f"{gp * 1e9 / (148 * mhz * 1e6):.3f} pairs/SM/clk", flush=True)
