#!/usr/bin/env python
"""Write tests/golden/fig7_sweep.csv from oracle.fig7 (the only source of its values)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import fig7  # noqa: E402

with open(os.path.join(ROOT, "tests", "golden", "fig7_sweep.csv"), "w") as f:
    f.write(fig7.to_csv(fig7.sweep()))
