"""CPU: the host decoders of the narrow device-to-host deliveries
(paper_2009_03707_b200/csrc/host_decode.hpp: SSE2 byte-step prefix decode of the arc
sources, non-temporal widening of the multiplicities) against scalar restatements."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_host_decoders(tmp_path):
    exe = tmp_path / "host_decode_check"
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "paper_2009_03707_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "host_decode_check.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "host decoders ok" in out.stdout
