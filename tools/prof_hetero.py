"""Profiling driver: C3 hetero SAGE layer (bf16 W), 2 calls after warm-up (use under ncu)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import bench_configs as bc  # noqa: E402

bc.timed = lambda fn, reps=10, warm=3: [fn() for _ in range(warm + 2)] and 0.0
bc.mag_layer()
