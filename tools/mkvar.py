"""Build an experiment variant of the library: python tools/mkvar.py NAME [-DFLAG=V ...]
-> tools/variants/lib_NAME.so (timed by tools/variants/run.sh NAME ...)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_05885_b200.build import build  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
root = os.path.join(os.path.dirname(os.path.abspath(__file__)), "variants")
print(build(extra=flags, force=True, out=os.path.join(root, f"lib_{name}.so"), build_dir=f"/tmp/jzvar/_b_{name}"))
