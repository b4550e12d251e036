"""Build liblag.so from the csrc/ of a git revision (A/B timing of a change
on one box).  usage: python scripts/build_rev.py REV OUT.so"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2004_02003_b200 import build as B  # noqa: E402


def main(rev, out):
    tmp = tempfile.mkdtemp()
    tar = subprocess.run(["git", "-C", ROOT, "archive", rev, "paper_2004_02003_b200/csrc", "include"],
                         check=True, capture_output=True).stdout
    subprocess.run(["tar", "-x", "-C", tmp], input=tar, check=True)
    B.CSRC = os.path.join(tmp, "paper_2004_02003_b200", "csrc")
    if hasattr(B, "INCLUDE"):
        B.INCLUDE = os.path.join(tmp, "include")
    print(B.build(out=os.path.abspath(out)))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
