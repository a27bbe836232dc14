"""Build experiment variants of libkdfused.so (timing A/B only; never the product): name=DEFINE[,DEFINE...]

    python scripts/build_variants.py gv4=KD_X_GV4 nog=KD_X_NOGSTORE nost=KD_X_NOSTAGE
-> paper_2603_01875_b200/libkdfused_<name>.so, selected at run time with KD_LIB_PATH."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_01875_b200 import build as B  # noqa: E402

for arg in sys.argv[1:]:
    name, defs = arg.split("=", 1)
    print(B.build(force=True, defines=tuple(defs.split(",")), out=os.path.join(B.HERE, f"libkdfused_{name}.so")))
