"""The runner's merged kernel sequences against their unmerged forms.

ops.cu merges steps by linearity of the NTT (ModDown with the following
rescale, the top-limb INTT, rotate-and-accumulate with one ModDown NTT per
output limb).  Each merge has an environment switch back to the plain
sequence (read once per process), so every combination is run in its own
process on the same seeded product and must give the same ciphertext bits.
HS_NO_GROUP_ROT turns off the per-key-group ModUp/inner product of the
accumulation rotations, HS_KSI_LDG the bulk-async inner-product kernel,
HS_ALIGN_MAX=3 runs the pair list in ranges of at most 3 aligned operands
(the path large configs take when the aligned operands exceed HBM), and
HS_NTT_F64=0 keeps every forward NTT on the integer (Shoup) butterflies
instead of the FP64-pipe butterflies used for ~50-bit primes.
The default path itself is checked against the oracle and the golden
vectors in test_gpu_parity.py.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[2])
import numpy as np
import paper_2604_11659_b200 as P
from helpers import digest
from test_gpu_parity import product_runner_case, _arr
out = {}
for (n, sb, L, seed, dim, sp, mseed) in [(8192, 45, 4, 2024, 12, 0.6, 5), (16384, 50, 2, 2024, 16, 0.7, 3)]:
    res = product_runner_case(P, n, sb, L, seed, dim, sp, mseed)[7]
    out[f"{n}_{L}"] = digest(_arr(res.ctxt))
print("DIGESTS " + json.dumps(out))
"""

SWITCHES = ["HS_SPLIT_MODDOWN_RESCALE", "HS_TOPLIMB_FWD", "HS_SPLIT_ROTATE_ACCUM", "HS_NO_GROUP_ROT",
            "HS_KSI_LDG", "HS_ALIGN_MAX", "HS_NTT_F64"]
VALUES = {"HS_ALIGN_MAX": "3", "HS_NTT_F64": "0"}     # 3 aligned operands per range; integer butterflies


def _digests(env_on):
    env = dict(os.environ)
    for k in SWITCHES:
        env.pop(k, None)
    for k in env_on:
        env[k] = VALUES.get(k, "1")
    p = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, os.path.join(ROOT, "tests")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    line = next(x for x in p.stdout.splitlines() if x.startswith("DIGESTS "))
    return json.loads(line[len("DIGESTS "):])


def test_merged_sequences_equal_plain_sequences():
    base = _digests([])
    for on in (["HS_SPLIT_MODDOWN_RESCALE"], ["HS_TOPLIMB_FWD"], ["HS_SPLIT_ROTATE_ACCUM"],
               ["HS_NO_GROUP_ROT"], ["HS_KSI_LDG"], ["HS_ALIGN_MAX"], ["HS_NTT_F64"], SWITCHES):
        assert _digests(on) == base, on
