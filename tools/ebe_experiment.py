"""Runs the expected-barycenter-effect experiment (bench.cpp:483-540 defaults) on the device."""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_2211_00805_b200 import knn_bench as kb  # noqa: E402

t0 = time.perf_counter()
res = kb.ebe_experiment(kb.EbeConfig())
print(json.dumps({"tau": res["tau"].tolist(), "tau_tv": res["tau_tv"].tolist(), "treatment_shift": 5.0,
                  "graph_size": res["graph_size"], "converged": [res["converged_treated"],
                                                                  res["converged_control"]],
                  "seconds": time.perf_counter() - t0}))
