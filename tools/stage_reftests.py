"""Stage the reference's own fp64 unit tests for tests/test_gpu_reference_suite.py.

Copies R/pkg/tests/{conftest,test_convolution,test_distance,test_derivatives,
test_sign}.py and the test-geometry module R/pkg/src/eikfld/shapes.py into
oracle/_ref/reftests/ (git-ignored, like the rest of oracle/_ref: it travels
to the GPU box with the working tree but never enters the history).  Run by
__graft_entry__.build() when /root/reference is present; the GPU box only
uses the staged copy.
"""

import hashlib
import os
import shutil
import sys

REF = "/root/reference/pkg"
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DST = os.path.join(REPO, "oracle", "_ref", "reftests")


def stage() -> bool:
    if not os.path.isdir(REF):
        return False
    os.makedirs(DST, exist_ok=True)
    names = ["conftest.py", "test_convolution.py", "test_distance.py", "test_derivatives.py", "test_sign.py"]
    lines = []
    for n in names:
        shutil.copyfile(os.path.join(REF, "tests", n), os.path.join(DST, n))
        lines.append(n)
    shutil.copyfile(os.path.join(REF, "src", "eikfld", "shapes.py"), os.path.join(DST, "shapes.py"))
    lines.append("shapes.py")
    with open(os.path.join(DST, "MANIFEST"), "w") as f:
        for n in lines:
            h = hashlib.sha256(open(os.path.join(DST, n), "rb").read()).hexdigest()
            f.write(f"{h}  {n}\n")
    return True


if __name__ == "__main__":
    ok = stage()
    print("staged" if ok else "reference not present; nothing staged", DST)
    sys.exit(0)
