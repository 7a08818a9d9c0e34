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


def test_oracle_extensions_pinned():
    """Relativistic (n_body_1pn) and hot-start extensions of the oracle: Schwarzschild
    limit, perihelion advance, PC vs RKF7(8), Chebyshev velocities, hot-start fixed point
    (oracle/ext_tests.cpp; the reference has no such path)."""
    build()
    exe = os.path.join(os.path.dirname(KAT), "ext_tests")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    lines = r.stdout.strip().splitlines()
    assert r.returncode == 0, "\n".join(l for l in lines if l.startswith("FAIL"))
    summary = lines[-1].split()
    assert summary[0] == "SUMMARY" and int(summary[2]) == 0 and int(summary[1]) >= 7
