"""Runs the paper's kNN distance-ranking benchmark (bench.cpp:246-371 defaults) on the device."""
import json
import sys

sys.path.insert(0, ".")
from paper_2211_00805_b200 import knn_bench as kb  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
seeds = [int(s) for s in args] or [1, 2, 3]
methods = (["geodesic_sinkhorn", "dense_sinkhorn_w1", "dense_sinkhorn_w2"]
           + (["euler_sinkhorn"] if "--euler" in sys.argv else []))
res = kb.knn_benchmark(kb.KnnBenchConfig(seeds=seeds, methods=methods,
                                         no_stagnation_abort="--no-stagnation-abort" in sys.argv))
for m in methods:
    iters = [max(s["iterations"][m]) for s in res["per_seed"]]
    print(json.dumps({"method": m, "seeds": seeds, "max_iterations": iters, **res["mean_report"][m]}))
