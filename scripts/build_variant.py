"""Build a variant of libzs.so with extra -D defines: build_variant.py NAME -DX=1 ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_17435_b200 import build as b  # noqa: E402
name, defs = sys.argv[1], sys.argv[2:]
print(b.build(force=True, verbose=False, defines=defs, lib=os.path.join(b.PKG, f"libzs_{name}.so")))
