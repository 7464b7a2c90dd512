"""Print the SASS of one kernel from a .so: python tools/sass_fn.py LIB PATTERN"""
import re
import subprocess
import sys

lib, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
blocks = re.split(r"\n\s*Function : ", out)
for b in blocks[1:]:
    name = b.split("\n", 1)[0].strip()
    if re.search(pat, name):
        print("Function:", name)
        print(b.split("\n", 1)[1])
        break
