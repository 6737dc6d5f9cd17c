"""CPU: the header-only C++ wrapper (include/tagdsp_gpu.hpp) compiles a
reference-style caller (examples/detect_recording_gpu.cpp) and links against
libtagdsp_gpu.so; the binary runs its no-GPU path."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_wrapper_compiles_links_and_runs(tmp_path):
    exe = tmp_path / "drg"
    libdir = os.path.join(ROOT, "paper_2005_10445_b200")
    cmd = ["g++", "-std=c++20", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "detect_recording_gpu.cpp"), "-L" + libdir, "-ltagdsp_gpu",
           "-Wl,-rpath," + libdir, "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stderr
    assert "870912" in out.stdout
