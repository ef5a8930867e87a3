"""Raw NVML clock-event masks and nvidia-smi reasons during a sustained GEMM loop."""
import subprocess
import threading
import time

import pynvml
import torch

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
dev = torch.device("cuda", 0)
a = torch.randn(8192, 8192, device=dev).bfloat16()
b = torch.randn(8192, 8192, device=dev).bfloat16()
masks, errs, clocks = [], [], []
stop = threading.Event()


def sample():
    while not stop.is_set():
        try:
            clocks.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            masks.append(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))
        time.sleep(0.01)


smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                        "clocks_event_reasons.active,clocks_event_reasons.sw_power_cap,"
                        "clocks_event_reasons.hw_slowdown", "--format=csv", "-lms", "200"],
                       stdout=subprocess.PIPE, text=True)
th = threading.Thread(target=sample)
th.start()
t0 = time.time()
while time.time() - t0 < 3.0:
    for _ in range(20):
        torch.matmul(a, b)
    torch.cuda.synchronize()
stop.set()
th.join()
smi.terminate()
out = smi.communicate()[0]
print("nvml masks (hex, unique):", sorted({hex(m) for m in masks}), "errors:", errs[:3])
print("clocks median", sorted(clocks)[len(clocks) // 2])
print("nvidia-smi:\n" + "\n".join(out.splitlines()[:12]))
