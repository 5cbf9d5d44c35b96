"""The reference's own engine test suite (pkg/tests/test_engine.py,
test_encmat.py) run against the drop-in: ``hespmm.engine``'s CSR/C runner
is replaced by ``ReferenceBridge`` (tests/ref_bridge_plugin.py; its device
half is the CPU oracle in this GPU-less container).  Every reference
assertion -- plaintext agreement, op-count laws, rotation predictor,
methods agreeing pairwise, errors -- must hold.  Build container only (the
reference does not exist on the GPU box)."""

import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

pytestmark = pytest.mark.skipif(not os.path.isdir("/root/reference/pkg"),
                                reason="the reference package is only in the build container")


def test_reference_engine_suite_through_the_bridge():
    sys.path.insert(0, os.path.join(HERE, "golden"))
    from make_golden import SCRATCH, ref_import
    ref_import()                     # builds the reference's Cython kernels in /tmp
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(SCRATCH, "src"), HERE, ROOT,
                                         env.get("PYTHONPATH", "")])
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "ref_bridge_plugin",
                        "-p", "no:cacheprovider", os.path.join(SCRATCH, "tests", "test_engine.py"),
                        os.path.join(SCRATCH, "tests", "test_encmat.py")],
                       cwd=SCRATCH, env=env, capture_output=True, text=True, timeout=1200)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]
    assert " passed" in p.stdout
    calls = int(p.stdout.split("REF_BRIDGE_CALLS")[1].split()[0])
    assert calls >= 10, calls         # the reference's tests really went through the bridge
