"""Every environment tunable the library reads is documented in include/nw.h (the boundary's
contract lists them as performance-only switches)."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_env_tunable_is_documented():
    csrc = os.path.join(ROOT, "paper_2102_13272_b200", "csrc")
    used = set()
    for f in os.listdir(csrc):
        if f.endswith((".cu", ".cuh", ".h")):
            used |= set(re.findall(r'(?:getenv|env_int)\("(NW_[A-Z0-9_]+)"', open(os.path.join(csrc, f)).read()))
    header = open(os.path.join(ROOT, "include", "nw.h")).read()
    assert used, "no tunables found"
    missing = sorted(v for v in used if v not in header)
    assert not missing, missing
