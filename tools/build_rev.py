"""Build the library of another git revision as an A/B variant:

    python tools/build_rev.py HEAD headlib   ->  paper_1408_1605_b200/build/variants/libheadlib.so

(the revision's csrc/ and include/ are exported to /tmp with `git archive`, then compiled with
the current build flags)."""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1408_1605_b200 import _build  # noqa: E402

rev, name = sys.argv[1], sys.argv[2]
d = tempfile.mkdtemp(prefix=f"bfs200_{name}_")
tar = subprocess.run(["git", "-C", ROOT, "archive", rev, "paper_1408_1605_b200/csrc", "include"], check=True,
                     capture_output=True).stdout
subprocess.run(["tar", "-x", "-C", d], input=tar, check=True)
print(_build.build_variant(name, [], force=True, csrc=os.path.join(d, "paper_1408_1605_b200", "csrc"),
                           include=os.path.join(d, "include")))
