"""Mutation check of the oracle's pins.

oracle.c carries MUT(k) hooks, each one plausible bug; CX_ORACLE_MUTATION=k
builds a separate liboracle_mut{k}.so with that bug. For every k the oracle pin
suite (worked examples, closed forms, library equivalences, mpmath brute force)
must FAIL -- otherwise the pins could not see that mistake."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PIN_TESTS = ["tests/test_oracle_golden.py", "tests/test_oracle_forward.py",
             "tests/test_oracle_linearize.py"]

MUTATIONS = {
    1: "TreeLSTM forget gate computed on h~ instead of each child h_k",
    2: "MV-RNN operands paired [A a; B b] instead of [B a; A b]",
    3: "TreeGRU update gate swapped: (1 - z) h~ + z g",
    4: "MV-RNN W_M multiplies the transposed child matrices",
    5: "TreeGRU reset gate applied to h~ instead of per child",
    6: "TreeFC halves swapped: W[:, :H] multiplies h_right",
    7: "DAG-RNN internal nodes drop the input projection W_x x",
    8: "TreeLSTM leaf memory cell uses sigma(u) instead of tanh(u)",
    9: "linearization: descending input id inside a level",
    10: "linearization: level_begin numbered leaves-first",
    11: "SimpleTreeGRU keeps the z * h~ term",
    12: "MV-RNN B a computed as B^T a",
    13: "TreeLSTM forget gate f_k multiplies another child's c",
    14: "TreeGRU leaf h = z * g instead of (1 - z) * g",
}


def _run(k):
    # the mutated oracle must build (a compile error would also fail the pins)
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        b = subprocess.run(["gcc", "-std=c99", "-O2", "-fPIC", "-shared", "-Wall", "-Werror",
                            f"-DCX_ORACLE_MUTATION={k}", "-o", os.path.join(d, "m.so"),
                            os.path.join(ROOT, "oracle", "oracle.c"), "-lm"],
                           capture_output=True, text=True)
        if b.returncode != 0:
            return k, -1, b.stderr[-400:]
    env = dict(os.environ, CX_ORACLE_MUTATION=str(k))
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    p = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        "-m", "not gpu"] + PIN_TESTS, cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    return k, p.returncode, p.stdout[-400:]


def test_every_mutation_fails_a_pin():
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        res = list(ex.map(_run, sorted(MUTATIONS)))
    survivors = [(k, MUTATIONS[k], out) for k, rc, out in res if rc != 1]
    assert not survivors, f"mutations not caught by any pin: {survivors}"
