"""Diagnostic: mp_worker's body with 8 in-process ranks on one GPU, full traceback on failure."""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1710_06952_b200 as P
import mp_worker

world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
tg = P.ThreadGroup(world)
try:
    fails = P.run_ranks(world, lambda r: mp_worker.body(r, world, 0, mp_worker.ThreadRanks(tg, r)), group=tg)
    print("FAILS:", fails[0])
except BaseException:
    traceback.print_exc()
    print("EXCEPTION")
