"""Build tuning variants of libmpcd into build/variants/ (one .so per -D set).

    python tools/build_variants.py NAME:DEF1,DEF2 NAME2:DEF ...
Then on the GPU: MPCD_LIB=build/variants/NAME.so python bench.py ...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_11878_b200 import _build  # noqa: E402

OUT = os.path.join(_build.ROOT, "build", "variants")

if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    for spec in sys.argv[1:]:
        name, _, defs = spec.partition(":")
        path = _build.build(force=True, defines=[d for d in defs.split(",") if d],
                            out=os.path.join(OUT, name + ".so"))
        print(path)
