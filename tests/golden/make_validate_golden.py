"""Reference validator verdicts on the committed fixtures and their corruptions.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_validate_golden.py

Writes tests/golden/validate_cases.json: {case: violations} from the UNMODIFIED
reference `bbox.validate_file` (format.py:476-548)."""

import json
import sys
import tempfile
from pathlib import Path

from bbox import validate_file

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
from corruptions import ARRAY_RECIPES, FIXTURES, RECIPES  # noqa: E402


def main():
    out = {}
    with tempfile.TemporaryDirectory() as td:
        for fx in FIXTURES:
            raw = (HERE / f"{fx}.bbox").read_bytes()
            cases = {"clean": lambda b: b, **RECIPES}
            if fx.startswith("mixed"):
                cases.update(ARRAY_RECIPES)
            for name, fn in cases.items():
                p = Path(td) / f"{fx}_{name}.bbox"
                p.write_bytes(fn(raw))
                out[f"{fx}/{name}"] = validate_file(p).violations
    (HERE / "validate_cases.json").write_text(json.dumps(out, indent=1))
    print(len(out), "cases")


if __name__ == "__main__":
    main()
