"""The drop-in's exceptions are the reference's classes when gmodelc is importable
(refexec.py:35, intrinsics.py:16-24, partition.py:18-30)."""

import subprocess
import sys
from pathlib import Path

import pytest

REF_SRC = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[1]

pytestmark = pytest.mark.skipif(not REF_SRC.exists(), reason="reference sources only in the build container")

PROBE = r"""
import sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {ref!r})
import gmodelc.refexec as rx, gmodelc.intrinsics as ri, gmodelc.partition as rp
from paper_1105_4424_b200 import executor, intrinsics, partition
assert issubclass(executor.MissingBinding, rx.MissingBinding) and issubclass(executor.MissingBinding, KeyError)
e = intrinsics.UnknownIntrinsic("top/t", "nope")
assert isinstance(e, ri.UnknownIntrinsic) and e.op_name == "nope" and "nope" in str(e)
assert issubclass(intrinsics.IntrinsicShapeMismatch, ri.IntrinsicShapeMismatch)
u = partition.UnallocatedTask("top/t")
assert isinstance(u, rp.UnallocatedTask) and u.task_path == "top/t"
assert issubclass(partition.MissingGeometry, rp.MissingGeometry)
assert issubclass(partition.CyclicTaskGraph, rp.CyclicTaskGraph)
try:
    raise executor.MissingBinding("p_x")
except rx.MissingBinding:
    pass
print("ok")
"""

PROBE_NO_REF = r"""
import sys
sys.path.insert(0, {root!r})
from paper_1105_4424_b200 import executor, intrinsics, partition
assert executor.MissingBinding.__mro__[1] is KeyError
assert intrinsics.UnknownIntrinsic("a", "b").op_name == "b"
assert partition.UnallocatedTask("t").task_path == "t"
print("ok")
"""


def _run(code):
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip().endswith("ok")


def test_exceptions_derive_from_reference_classes():
    _run(PROBE.format(root=str(ROOT), ref=str(REF_SRC)))


def test_exceptions_without_reference_keep_builtin_bases():
    _run(PROBE_NO_REF.format(root=str(ROOT)))
