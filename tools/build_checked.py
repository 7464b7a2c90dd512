"""Build the checked library (SB_CHECKED: bounds traps + hand-off timing perturbation)
into checked/libsliceblur_b200.so (git-ignored, travels to the GPU box).

    python tools/build_checked.py
    SB_LIB_PATH=checked/libsliceblur_b200.so python tools/checked_run.py --check ...
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1107_4958_b200 import build as b  # noqa: E402

d = os.path.join(ROOT, "checked")
os.makedirs(d, exist_ok=True)
b.OUT = os.path.join(d, "libsliceblur_b200.so")
b.STAMP = b.OUT + ".flags"
os.environ["SB_NVCC_EXTRA"] = "-DSB_CHECKED=1"
orig_join = os.path.join


def join(*a):
    if len(a) == 2 and a[0] == b.PKG and a[1] == "build_obj":
        return orig_join(d, "obj")
    return orig_join(*a)


os.path.join = join
print(b.build(force="--force" in sys.argv))
