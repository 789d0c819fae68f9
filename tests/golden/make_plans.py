#!/usr/bin/env python3
"""Generate tests/golden/packing_plans.json: the reference's make_packing_plan
(proj/include/lrbatch/plan.hpp:66-100) for each of its machine models and
every rank 1..128, captured through oracle/_ref (which resolves the machine
files from /root/reference). The GPU box has no /root/reference, so the
reference's packed drivers (packed_multiply, blr_matvec) replay these plans
there — the plan is the reference's own output, not a re-derivation.

    python tests/golden/make_plans.py        # needs /root/reference and `make ref`
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

MACHINES = ("epyc-7502", "skylake-x-6148", "a64fx")


def main():
    if not O.ref_machines_available():
        sys.exit("needs /root/reference (the machine files)")
    out = {"generator": "tests/golden/make_plans.py", "fields": list(O.PLAN_FIELDS),
           "source": "make_packing_plan(resolve_machine(m), rank, 0) via oracle/_ref",
           "plans": {}}
    for m in MACHINES:
        out["plans"][m] = {str(r): O.ref_packing_plan_live(m, r) for r in range(1, 129)}
    path = os.path.join(ROOT, "tests", "golden", "packing_plans.json")
    with open(path, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
        fh.write("\n")
    print(f"wrote {path}")


if __name__ == "__main__":
    main()
