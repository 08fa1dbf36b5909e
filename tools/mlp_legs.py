"""Config-3 (MLP) bench legs on their own: replay, free-running 8 ranks on one GPU, GEMM sweep."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch

import bench
import synth
import paper_1710_06952_b200 as P
import gemm_sweep
import mlp_free_running_1gpu

out = {"mlp_config3": bench.mlp_leg(P, synth, torch)}
print(json.dumps(out), flush=True)
out["mlp_config3_free_running_1gpu"] = mlp_free_running_1gpu.run(8)
print(json.dumps(out["mlp_config3_free_running_1gpu"]), flush=True)
out["mlp_gemm_sweep"] = gemm_sweep.sweep(reps=10)
print(json.dumps(out))
