"""Fetch the reference package's own test suite for tests/ref_suite.

TEST INFRASTRUCTURE (build container only): copies the reference's
pkg/tests/test_*.py and its synthetic test-image generator
pkg/src/blockmend/corpus.py (test data, out of the path's scope) from
/root/reference into tests/ref_suite/_ref/.  `_ref/` is git-ignored (the
reference's sources never enter this repository's history) but not
gpurun-ignored, so the suite travels to the GPU box, where
tests/ref_suite/conftest.py runs it against this package.  Run by
__graft_entry__.build() when /root/reference is present.
"""

import glob
import os
import shutil

HERE = os.path.dirname(os.path.abspath(__file__))
DEST = os.path.join(HERE, "_ref")
REFERENCE = "/root/reference/pkg"


def fetch(reference: str = REFERENCE) -> bool:
    tests = sorted(glob.glob(os.path.join(reference, "tests", "test_*.py")))
    corpus = os.path.join(reference, "src", "blockmend", "corpus.py")
    if not tests or not os.path.exists(corpus):
        return False
    os.makedirs(DEST, exist_ok=True)
    for src in tests + [corpus]:
        dst = os.path.join(DEST, os.path.basename(src) if src != corpus else "ref_corpus.py")
        shutil.copyfile(src, dst)
    return True


if __name__ == "__main__":
    print("fetched" if fetch() else "reference suite not found")
