"""The CPU oracle is pinned to the reference's own known-answer tests and
properties (oracle/kat_tests.cpp restates proj/tests/*.cpp + acceptance.cpp)."""
import os
import subprocess

from oracle.oracle_py import KAT, build


def test_oracle_passes_reference_kats():
    build()
    r = subprocess.run([KAT], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    lines = r.stdout.strip().splitlines()
    assert r.returncode == 0, "\n".join(l for l in lines if l.startswith("FAIL"))
    summary = lines[-1].split()
    assert summary[0] == "SUMMARY" and int(summary[2]) == 0 and int(summary[1]) >= 85
