"""GPU rows in the reference's results schema: round trip through our writer
and the reference's own csv.hpp reader/validator (oracle/_ref), CPU only."""
import ctypes
import math
import os

import pytest

import oracle
from paper_2507_20173_b200 import records
from paper_2507_20173_b200.__main__ import main as cli_main


def _ref_reader():
    if not os.path.exists(oracle.REF_SO) and not os.path.isdir(oracle.REF_INCLUDE):
        pytest.skip("reference not available")
    L = oracle.Reference().L
    L.ref_read_csv.restype = ctypes.c_int
    L.ref_read_csv.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int), ctypes.c_char_p, ctypes.c_int]
    return L


def sample_records():
    return [
        records.BenchRecord("custom", 1, "graph", 10_000_000, "gpu", 0, 10_000_000, 100, 0.0131, 0.0, 0xDD7AF4C450353D19),
        records.BenchRecord("gpu-persistent", 1, "cluster", 4096, "gpu", 3, 4096, 100000, 0.143, 0.0, 0x5AA6CA83B4825C14),
        records.BenchRecord("gpu-stream", 8, "graph", 125_000_000, "gpu", 1, 10**9, 20, math.nan, math.nan, 0),
    ]


def test_write_read_roundtrip():
    text = records.write_csv_string(sample_records())
    assert text.splitlines()[0] == records.CSV_HEADER
    back = records.read_csv(text)
    assert len(back) == 3 and back[0].checksum == 0xDD7AF4C450353D19 and back[2].failed()
    assert records.format_seconds(0.1) == "0.1" and records.format_seconds(math.nan) == "NaN"


def test_reference_reader_accepts_gpu_rows():
    L = _ref_reader()
    text = records.write_csv_string(sample_records()).encode()
    issues = ctypes.c_int(-1)
    err = ctypes.create_string_buffer(256)
    n = L.ref_read_csv(text, ctypes.byref(issues), err, 256)
    assert n == 3, err.value
    assert issues.value == 0
    bad = b"experiment,threads\n1,2\n"
    assert L.ref_read_csv(bad, ctypes.byref(issues), err, 256) == -1
    assert b"unknown header" in err.value


def test_cli_usage_errors_exit_2(capsys):
    assert cli_main(["simulate", "--fish", "notanumber"]) == 2
    assert cli_main(["nosuchcommand"]) == 2
