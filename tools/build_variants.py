"""Build libucp_b200 variants with extra -D macros into variants/<name>.so
(experiments: `UCP_B200_LIB=variants/<name>.so python ...`).

    python tools/build_variants.py name1:MACRO=1,OTHER=2 name2:...
"""
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1908_04489_b200 import _build  # noqa: E402


def one(spec):
    name, _, macros = spec.partition(":")
    out = ROOT / "variants" / f"{name}.so"
    out.parent.mkdir(exist_ok=True)
    _build.build(force=True, lib=out, defines=tuple(m for m in macros.split(",") if m))
    return str(out)


if __name__ == "__main__":
    with ThreadPoolExecutor(4) as ex:
        for p in ex.map(one, sys.argv[1:]):
            print(p)
