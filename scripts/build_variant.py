"""Build an experiment variant of the library next to the product build:
    python scripts/build_variant.py NAME [-DMACRO=VALUE ...]
-> _abtest/libNAME.so (objects in _abtest/obj_NAME); select it at run time with
NUFFT_B200_LIB=$PWD/_abtest/libNAME.so (paper_1701_04492_b200/_lib.py)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
name, extra = sys.argv[1], sys.argv[2:]
os.environ["NB_NVCC_EXTRA"] = " ".join(extra)
from paper_1701_04492_b200 import build_ext  # noqa: E402

ab = os.path.join(ROOT, "_abtest")
os.makedirs(ab, exist_ok=True)
build_ext.OBJ = os.path.join(ab, "obj_" + name)
build_ext.LIB = os.path.join(ab, f"lib{name}.so")
build_ext._build_example = lambda: None
print(build_ext.build())
