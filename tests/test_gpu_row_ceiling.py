"""hbk_row_ceiling, the hardware anchor bench.py reports beside the HBM
roofline (roofline.gather.hardware): argument checks, and one small launch
timed on the caller's stream gives a finite, positive row rate."""
from __future__ import annotations

import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


def test_row_ceiling_launch_and_guards():
    import torch

    from paper_1904_03329_b200 import _native as N

    N.require_device()
    with pytest.raises(ValueError):
        N.call("hbk_row_ceiling", C.c_int64(1000), 3, C.c_int64(1 << 20), N.stream_ptr())  # not 2^k
    with pytest.raises(ValueError):
        N.call("hbk_row_ceiling", C.c_int64(1024), 0, C.c_int64(1 << 20), N.stream_ptr())
    N.call("hbk_row_ceiling", C.c_int64(1 << 12), 3, C.c_int64(1 << 22), N.stream_ptr())
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    N.call("hbk_row_ceiling", C.c_int64(1 << 12), 3, C.c_int64(1 << 22), N.stream_ptr())
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    assert 0 < ms < 1000
    groups = 3 * torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count * 32
    rows = groups * max(8, ((1 << 22) // groups + 7) // 8 * 8)
    assert rows / (ms * 1e-3) > 1e9  # well above a billion rows/s on any B200
    N.call("hbk_row_ceiling", C.c_int64(0), 1, C.c_int64(1), N.stream_ptr())  # frees the scratch
    N.call("hbk_row_ceiling", C.c_int64(1 << 10), 1, C.c_int64(1 << 16), N.stream_ptr())  # re-allocates
    torch.cuda.synchronize()


def test_row_ceiling_stream_needs_the_matrix_and_runs():
    import torch

    from paper_1904_03329_b200 import _native as N

    N.require_device()
    rows = 1 << 12
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    n = 4 * sms * 32 * 64
    idx = torch.randint(0, rows, (n,), device="cuda", dtype=torch.int32)
    N.call("hbk_row_ceiling", C.c_int64(0), 1, C.c_int64(1), N.stream_ptr())  # no matrix now
    with pytest.raises(ValueError):
        N.call("hbk_row_ceiling_stream", C.c_void_p(idx.data_ptr()), C.c_int64(n), C.c_int64(rows), 4,
               N.stream_ptr())
    N.call("hbk_row_ceiling", C.c_int64(rows), 4, C.c_int64(1 << 16), N.stream_ptr())
    with pytest.raises(ValueError):  # too short for the grid
        N.call("hbk_row_ceiling_stream", C.c_void_p(idx.data_ptr()), C.c_int64(64), C.c_int64(rows), 4,
               N.stream_ptr())
    N.call("hbk_row_ceiling_stream", C.c_void_p(idx.data_ptr()), C.c_int64(n), C.c_int64(rows), 4,
           N.stream_ptr())
    torch.cuda.synchronize()
