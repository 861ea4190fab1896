"""Golden results of the reference window search (ringmpc search.py:159-334) on its desk CNN.

Runs the REFERENCE package only; writes tests/golden/golden_search.json (committed):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_search_golden.py
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))  # tests/ for golden_cases

from ringmpc import models, search  # noqa: E402  (reference package)

import golden_cases as gc  # noqa: E402


def main():
    out = {}
    for case in gc.SEARCH_CASES:
        model = models.build_cnn(11)
        x_f, labels = gc.search_inputs(case)
        if case["kind"] == "eco":
            res = search.search_eco(model, x_f, labels, seed=case["seed"])
        else:
            res = search.search_budget(model, x_f, labels, case["budget"], threshold=case.get("threshold"),
                                       candidate_widths=tuple(case["widths"]), seed=case["seed"])
        out[case["name"]] = res.to_json()
        print(case["name"], json.dumps(out[case["name"]]))
    with open(os.path.join(HERE, "golden_search.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
