"""The bench's config-2 and config-1 legs on their own (tools, not the product)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import synth
import paper_1710_06952_b200 as P

c2 = bench.config2_leg(P, synth, torch)
c1 = bench.config1_leg(P, synth, torch)
print(json.dumps({k: round(v["gossip_steps_per_s"]) for k, v in c2.items() if isinstance(v, dict)}),
      json.dumps({k: round(v["us_per_event"], 2) for k, v in c1.items() if isinstance(v, dict)}))
