"""run_batched (engine.hpp:120-212) in the drop-in headers against the
reference's own template, on the same worker workload (oracle/
run_batched_probe.hpp): batching from adjust_batch_size, hooks, per-slot
errors, infeasible slots, timings and the fixed-order mean.  Host-only (no
GPU): tests/cpp/_build/facade_main's `batched` command vs oracle/_ref."""
import ctypes as C
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "facade_main")


@pytest.mark.parametrize("count,batch,threads,budget,per_bytes", [
    (1000, 128, 4, 2 << 30, 0),
    (257, 50, 3, 2 << 30, 8),
    (10, 1000, 1, 100, 64),        # budget below one scenario: batches of 1 + warning
    (3000, 1 << 20, 8, 4096, 16),  # budget-limited batches
    (1, 1, 2, 2 << 30, 0),
    (0, 16, 2, 2 << 30, 0),
])
def test_run_batched_matches_reference(reference, count, batch, threads, budget, per_bytes):
    if not os.path.exists(BIN):
        pytest.fail("tests/cpp/_build/facade_main not built (make -C paper_2602_05179_b200/csrc)")
    ours = subprocess.run([BIN, "batched", str(count), str(batch), str(threads), str(budget),
                           str(per_bytes)], capture_output=True, text=True, timeout=60)
    assert ours.returncode == 0, ours.stdout + ours.stderr
    buf = C.create_string_buffer(512)
    fn = reference.lib.ref_run_batched_probe
    fn.argtypes = [C.c_size_t, C.c_size_t, C.c_uint, C.c_ulonglong, C.c_ulonglong, C.c_char_p,
                   C.c_size_t]
    fn(count, batch, threads, budget, per_bytes, buf, 512)
    assert ours.stdout.strip() == buf.value.decode()
