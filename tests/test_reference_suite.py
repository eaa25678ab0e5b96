"""The reference's OWN test suite against the B200 engine (drop-in check).

Copies `/root/reference/pkg/tests` (all 11 files, 196 tests) into a temporary directory and
runs it twice in subprocesses: once unmodified, once with `integration/spectool_b200.install`
(the reference-side binding of INTEGRATION.md) swapping `spectool.engine.EngineSim` for
`B200Engine` before any test module imports it. The reference's own tokens, scripts, clients,
`EngineClient`, workload fleets and error classes drive the B200 engine; its runtime is the
host-only stub (`tests/stub_runtime.py`: same control decisions, no GPU), so this runs on CPU.

Pass criterion: the B200 run fails exactly the tests the unmodified reference fails in this
image (the matplotlib-only plot / criterion-9 tests: matplotlib is not installed). Skipped
where the reference is absent (the GPU box).
"""

import re
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg")
ROOT = Path(__file__).resolve().parent.parent

pytestmark = pytest.mark.skipif(not (REF / "tests").is_dir(), reason="reference tree not present")

PLUGIN = f'''
import sys
sys.path.insert(0, {str(ROOT)!r})
sys.path.insert(0, {str(ROOT / "tests")!r})
from integration import spectool_b200
from stub_runtime import StubRuntime
spectool_b200.install(lambda config: StubRuntime())
'''


def _run(tmp: Path, plugin: bool) -> tuple[int, set[str]]:
    args = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-o", "addopts=", str(tmp)]
    if plugin:
        args[3:3] = ["-p", "b200_plugin"]
    env = {"PYTHONPATH": f"{REF / 'src'}:{tmp}", "PATH": "/usr/bin:/bin", "HOME": str(tmp)}
    out = subprocess.run(args, cwd=tmp, env=env, capture_output=True, text=True, timeout=900).stdout
    failed = set(re.findall(r"^FAILED (\S+)", out, re.M))
    m = re.search(r"(\d+) passed", out)
    return (int(m.group(1)) if m else 0), failed


def test_reference_suite_on_b200_engine(tmp_path):
    dst = tmp_path / "tests"
    shutil.copytree(REF / "tests", dst)
    (dst / "b200_plugin.py").write_text(PLUGIN)
    ref_pass, ref_failed = _run(dst, plugin=False)
    b2_pass, b2_failed = _run(dst, plugin=True)
    assert b2_failed == ref_failed, (sorted(b2_failed - ref_failed), sorted(ref_failed - b2_failed))
    assert b2_pass == ref_pass and b2_pass >= 190, (b2_pass, ref_pass)
    # the only tests the unmodified reference fails here need matplotlib (absent from the image)
    assert all("plot" in t or "criterion_9" in t for t in ref_failed), ref_failed
    # the engine-facing files all pass on the B200 engine
    assert not any(t.split("::")[0] in ("test_engine.py", "test_orchestrator.py", "test_workload.py",
                                        "test_service.py") for t in b2_failed)
