"""A/B builds of the column-walker K1's compile-time shape into variants/ (git-ignored;
travels to the GPU box with the snapshot).  scripts/gpu_variants.sh benches each."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2306_12517_b200 import _build  # noqa: E402

VARIANTS = {a.split(":")[0]: tuple(x for x in a.split(":")[1].split(",") if x) for a in sys.argv[1:]}
(ROOT / "variants").mkdir(exist_ok=True)
for name, defs in VARIANTS.items():
    _build.build(force=True, defines=defs or ("BBX_VARIANT=1",), out=ROOT / "variants" / f"libbbx_{name}.so")
    print("built", name, defs)
