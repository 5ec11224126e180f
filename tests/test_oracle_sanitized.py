"""The oracle under AddressSanitizer + UndefinedBehaviorSanitizer (SURVEY.md Sec. 4
level 5): the same C sources built with -fsanitize=address,undefined (build.py
oracle-asan) run the oracle pins in a child process with libasan preloaded.  Any
out-of-bounds access, use of uninitialised heap, signed overflow or other UB report
aborts the child (-fno-sanitize-recover=all), failing this test."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _runtime(name):
    p = subprocess.run(["gcc", f"-print-file-name={name}"], capture_output=True, text=True)
    path = p.stdout.strip()
    return path if os.path.isabs(path) and os.path.exists(path) else None


@pytest.mark.slow
def test_oracle_pins_under_asan_ubsan():
    import build
    lib = build.build_oracle(sanitize=True)
    asan = _runtime("libasan.so")
    if asan is None:
        pytest.skip("libasan not available")
    env = dict(os.environ, W3D_ORACLE_LIB=lib, LD_PRELOAD=asan,
               ASAN_OPTIONS="detect_leaks=0:abort_on_error=1:halt_on_error=1",
               UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1")
    # the oracle pins (warp, noise, compose, window/gamma, occlusion, brute force) and
    # the resampling pins, minus the 1e6-sample statistics test (slow under ASan)
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
           os.path.join(ROOT, "tests", "test_oracle_pins.py"),
           os.path.join(ROOT, "tests", "test_oracle_resample.py"),
           "-k", "not statistics_1e6"]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT, timeout=900)
    tail = (out.stdout + out.stderr)[-3000:]
    assert out.returncode == 0, tail
    assert "ERROR: AddressSanitizer" not in tail and "runtime error" not in tail, tail


@pytest.mark.slow
def test_asan_build_is_live():
    """Positive control: the sanitized oracle aborts on a deliberate overrun (an input
    buffer one voxel short of the 16^3 it is declared as: the identity warp's last read
    lands in the allocation's redzone), so a clean run above means something."""
    import build
    lib = build.build_oracle(sanitize=True)
    asan = _runtime("libasan.so")
    if asan is None:
        pytest.skip("libasan not available")
    code = ("import ctypes, numpy as np, oracle as O\n"
            "L = O.lib()\n"
            "img = np.zeros(16 ** 3 - 1, np.float32); out = np.zeros((16, 16, 16), np.float32)\n"
            "A = np.eye(3, 4, dtype=np.float32)\n"
            "L.oracle_warp_volume(img.ctypes.data, None, O._dims((16, 16, 16)).ctypes.data,\n"
            "    A.ctypes.data, 0, ctypes.c_float(0), 0, None, out.ctypes.data, None,\n"
            "    O._dims((16, 16, 16)).ctypes.data)\n")
    env = dict(os.environ, W3D_ORACLE_LIB=lib, LD_PRELOAD=asan,
               ASAN_OPTIONS="detect_leaks=0:halt_on_error=1")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         cwd=ROOT, timeout=120)
    assert out.returncode != 0 and "AddressSanitizer: heap-buffer-overflow" in out.stderr
