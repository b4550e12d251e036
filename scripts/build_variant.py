"""Build an experiment variant of liblag.so from a patched copy of csrc/.

usage: python scripts/build_variant.py OUT.so 'old=>new' ['old=>new' ...]
Each 'old=>new' is a literal text substitution applied to every csrc file
(it must match at least once).  The product sources are not touched."""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2004_02003_b200 import build as B  # noqa: E402


def main(out, subs):
    tmp = tempfile.mkdtemp()
    dst = os.path.join(tmp, "csrc")
    shutil.copytree(B.CSRC, dst)
    for sub in subs:
        old, new = sub.split("=>", 1)
        hit = 0
        for f in os.listdir(dst):
            p = os.path.join(dst, f)
            s = open(p).read()
            if old in s:
                hit += s.count(old)
                open(p, "w").write(s.replace(old, new))
        if not hit:
            raise SystemExit(f"substitution not found: {old!r}")
    B.CSRC = dst
    print(B.build(out=os.path.abspath(out), verbose="-v" in os.environ.get("VARIANT_FLAGS", "")))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
