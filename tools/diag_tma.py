"""Diagnose the TMA input transform: run configurations in fresh processes with NW_DEBUG_SYNC=1."""
import json, os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
RUN = os.path.join(HERE, "..", "tests", "_variant_run.py")
cases = [
    ({"config": "c2k9", "N": 2, "H": 40, "W": 36, "Cin": 32, "Cout": 64, "m_o": 3}, {}),
    ({"config": "c2k9", "N": 2, "H": 40, "W": 36, "Cin": 32, "Cout": 64, "m_o": 3}, {"NW_INPUT_TMA": "0"}),
    ({"config": "c2k9", "N": 2, "H": 40, "W": 36, "Cin": 64, "Cout": 64, "m_o": 3}, {}),
    ({"config": "c2k9", "N": 2, "H": 40, "W": 36, "Cin": 32, "Cout": 64}, {}),
    ({"config": "c2k9", "N": 2}, {}),
    ({"config": "c2k9", "N": 8}, {}),
    ({"config": "c2k9", "N": 32}, {}),
]
for spec, env in cases:
    e = dict(os.environ, NW_DEBUG_SYNC="1", **env)
    r = subprocess.run([sys.executable, RUN, json.dumps(spec), "/tmp/y.npy"], env=e, capture_output=True, text=True)
    lines = [l for l in r.stderr.splitlines() if "[nw]" in l or "Error" in l][:4]
    print(json.dumps(spec), env, "rc", r.returncode, lines, flush=True)
