"""Runs only bench.py's post-processing section (BASELINE configs[3])."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
print(json.dumps(bench.postproc_bench(torch, 0, M=M)))
