"""The pins must FAIL when the oracle is wrong (task ③): three single-edit mistakes -- the two the round-1
review applied by hand (violation checking rows only; FGW objective without its (1 - alpha) factor) and the one
this round's sweep found alive (the sign of the (eps - tau) ln T term) -- are applied to a copy of oracle/ and
the pin suites run against it.  The full sweep (70 mutations, profiles/r02_oracle_mutations.log) is
`python scripts/mutate_oracle.py`."""

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_pins_kill_known_mutations():
    sel = "violation: rows only,fgw_objective: dropped (1 - alpha),entropic_gw: sign of the tau term"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "mutate_oracle.py"), "--only", sel, "--jobs", "3"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mutations 3, killed 3, survived 0, not applied 0" in r.stdout, r.stdout
