"""Golden records of the reference's verify.error_table (rigaeig v0.1.0).

Inputs: dense generalized eigenpairs (scipy eigh(K, M), driver gvd) of the
reference's own build_system for a few small cases; outputs: the reference's
ErrorRecords.  Run in the build container (it imports /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_verify_golden.py
"""
import json
import os

import numpy as np
import scipy.linalg

from rigaeig.assembly import build_system
from rigaeig.verify import error_table

CASES = [(1, 16, 3, 0, 10), (2, 8, 2, 0, 12), (2, 8, 3, 1, 20), (3, 4, 2, 0, 12)]
out = {"generator": "tests/golden/make_verify_golden.py", "cases": []}
for d, ne, p, lv, cnt in CASES:
    s = build_system(d, ne, p, lv)
    lam, X = scipy.linalg.eigh(s.K.csr.toarray(), s.M.csr.toarray(), driver="gvd")
    recs = error_table(lam[:cnt], X[:, :cnt], s)
    out["cases"].append({"d": d, "ne": ne, "p": p, "level": lv, "count": cnt,
                         "records": [{"position": r.position, "indices": list(r.indices), "ev": r.ev,
                                      "efl": None if np.isnan(r.efl) else r.efl, "diagonal": r.diagonal}
                                     for r in recs]})
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "verify_golden.json")
json.dump(out, open(path, "w"), indent=1)
print("wrote", path, sum(len(c["records"]) for c in out["cases"]), "records")
