"""Build a variant of the library with extra nvcc flags into exp/<name>/ (A/B experiments).

    python tools/build_variant.py NAME -DSB_FOO=1 ...
    SB_LIB_PATH=exp/NAME/libsliceblur_b200.so python bench.py ...
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1107_4958_b200 import build as b  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
d = os.path.join(ROOT, "exp", name)
os.makedirs(d, exist_ok=True)
b.OUT = os.path.join(d, "libsliceblur_b200.so")
b.STAMP = b.OUT + ".flags"
b.PKG_OBJ = d
os.environ["SB_NVCC_EXTRA"] = " ".join(extra)
orig_join = os.path.join


def join(*a):
    if len(a) == 2 and a[0] == b.PKG and a[1] == "build_obj":
        return orig_join(d, "obj")
    return orig_join(*a)


os.path.join = join
print(b.build(force=True))
