"""pytest plugin (debug): while a stream capture is active, line-trace the
executor and report the first source line after which the capture became
invalidated."""
import functools
import sys

import torch
from cuda.bindings import runtime as rt

from paper_2503_04771_b200 import executor

ACTIVE = rt.cudaStreamCaptureStatus.cudaStreamCaptureStatusActive
_done = [False]


def _status():
    s = torch.cuda.current_stream().cuda_stream
    return rt.cudaStreamGetCaptureInfo(s)[1]


orig = executor.run_gemm


@functools.wraps(orig)
def run_gemm(*a, **k):
    if _done[0] or _status() != ACTIVE:
        return orig(*a, **k)
    last = ["start"]

    def tracer(frame, event, arg):
        if _done[0]:
            return None
        if event in ("line", "return", "call"):
            st = _status()
            if st != ACTIVE:
                _done[0] = True
                print(f"\n### capture invalidated; previous event {last[0]}; now "
                      f"{frame.f_code.co_filename}:{frame.f_lineno} {event}", flush=True)
                sys.settrace(None)
                return None
            last[0] = f"{frame.f_code.co_filename}:{frame.f_lineno} {event} {frame.f_code.co_name}"
        return tracer

    sys.settrace(tracer)
    try:
        return orig(*a, **k)
    finally:
        sys.settrace(None)


executor.run_gemm = run_gemm
