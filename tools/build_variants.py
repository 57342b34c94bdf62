"""Build tuning variants of the CUDA library into variants/ (gitignored; they
travel to the GPU box with the snapshot).  usage: build_variants.py name=DEF1,DEF2 ..."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_27210_b200 import _build  # noqa: E402

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def one(spec):
    name, _, defs = spec.partition("=")
    out = os.path.join(REPO, "variants", f"lib_{name}.so")
    _build.build(force=True, out=out, defines=[d for d in defs.split(",") if d])
    return out


if __name__ == "__main__":
    os.makedirs(os.path.join(REPO, "variants"), exist_ok=True)
    with ThreadPoolExecutor(4) as ex:
        for p in ex.map(one, sys.argv[1:]):
            print(p)
