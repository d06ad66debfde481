"""Just bench.py's per-op benchmarks (configs 1-4) as one JSON object."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

print(json.dumps(bench.op_benchmarks(), indent=1))
