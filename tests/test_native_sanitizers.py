"""the host encoder and the CPU oracle under AddressSanitizer + UndefinedBehavior-
Sanitizer.  tests/native/asan_driver.cpp is compiled together with encode.cpp and df11_oracle.c
(-fsanitize=address,undefined, halt on the first report) and run over edge cases and random inputs of
every value format, geometry and LUT width; every library encoding must round-trip through the oracle's
D1 and D2."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None or shutil.which("gcc") is None, reason="needs gcc / g++")
def test_encoder_and_oracle_under_asan_ubsan(tmp_path):
    flags = ["-O1", "-g", "-fno-omit-frame-pointer", "-fsanitize=address,undefined", "-fno-sanitize-recover=all"]
    ora = tmp_path / "oracle.o"
    subprocess.check_call(["gcc", "-std=c99", *flags, "-c", os.path.join(ROOT, "oracle", "df11_oracle.c"), "-o", str(ora)])
    exe = tmp_path / "asan_driver"
    subprocess.check_call(["g++", "-std=c++17", *flags, "-pthread",
                           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "paper_2504_11651_b200", "csrc"),
                           os.path.join(ROOT, "tests", "native", "asan_driver.cpp"),
                           os.path.join(ROOT, "paper_2504_11651_b200", "csrc", "encode.cpp"), str(ora), "-o", str(exe)])
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=0", UBSAN_OPTIONS="print_stacktrace=1")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert "0 failures" in r.stdout
