"""The C-ABI without Python: examples/c_abi_client.c (plain C, gcc, linked
against libdssp_ps.so and cudart) creates a server, pushes and pulls through
include/dssp_ps.h exactly as a non-Python FFI would, and checks the result
bit for bit against server.py:37's fp32 rule; it also prints the per-call
latency of the bare C-ABI."""

import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_client_push_pull_bit_exact():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "examples")], check=True)
    out = subprocess.run([os.path.join(ROOT, "examples", "c_abi_client"), "272474", "100"],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "bit-exact" in out.stdout, out.stdout
    for ragged in ("1", "5", "1027"):
        r = subprocess.run([os.path.join(ROOT, "examples", "c_abi_client"), ragged, "5"],
                           capture_output=True, text=True, timeout=120)
        assert r.returncode == 0 and "bit-exact" in r.stdout, r.stdout + r.stderr
