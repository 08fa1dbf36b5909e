"""The bench's config-1 leg on its own (tools, not the product)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import synth
import paper_1710_06952_b200 as P

print(json.dumps(bench.config1_leg(P, synth, torch)))
