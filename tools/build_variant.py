"""Build an A/B variant of the CUDA library with extra preprocessor defines.

    python tools/build_variant.py NAME [DEFINE ...]   ->  build/variants/NAME.so
    XA_LIB_PATH=build/variants/NAME.so python tools/time_coarse.py
"""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
from paper_2503_03479_b200 import build  # noqa: E402

if __name__ == "__main__":
    name, defs = sys.argv[1], sys.argv[2:]
    out = pathlib.Path(__file__).resolve().parent.parent / "build" / "variants" / f"{name}.so"
    print(build.build(force=True, defines=defs, out=out))
