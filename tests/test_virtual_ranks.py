"""In-process ranks sharing ONE GPU (-m gpu, runs on a 1-GPU box).

comm_local contexts (include/adpsgd.h) driven by host threads run the same
bodies as the one-process-per-GPU tests (tests/mp_worker.py, tests/mp_super.py):
cross-rank engine replay and free-running with remote try-locks, cooperative
mailboxes and commit flags, host-driven steps with device tickets, the D-PSGD
halo, consensus and AllReduce collectives, the App. A wait-free loop and
super-learners -- with every rank's memory on cuda:0 and the
collectives as fixed-order in-process reductions (comm.h) instead of NCCL.
Each body replays the device event log through the oracle (P:458-479 replay,
reading R22 for super-learners) and returns rank 0's failures."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))

pytestmark = pytest.mark.gpu


def _virtual(world, body_of):
    import paper_1710_06952_b200 as P
    import mp_worker
    tg = P.ThreadGroup(world)
    fails = P.run_ranks(world, lambda r: body_of(r, mp_worker.ThreadRanks(tg, r)), group=tg)
    return fails[0]


@pytest.mark.parametrize("world", [2, 4])
def test_virtual_ranks_parity(world):
    """mp_worker's checks 1-9 (full-size bench workload included) with `world`
    in-process ranks on cuda:0."""
    import mp_worker
    fails = _virtual(world, lambda r, G: mp_worker.body(r, world, 0, G))
    assert not fails, fails


@pytest.mark.skipif(os.environ.get("ADPSGD_TEST_WORLD8") != "1",
                    reason="opt-in (ADPSGD_TEST_WORLD8=1, ~85 s): 8 in-process ranks, the N = 8 protocol on one GPU")
def test_virtual_ranks_parity_world8():
    """mp_worker's checks with 8 in-process ranks on cuda:0: the cross-rank protocol at the
    world size the 8-GPU scaling run uses (this pool's boxes have at most 4 GPUs)."""
    import mp_worker
    fails = _virtual(8, lambda r, G: mp_worker.body(r, 8, 0, G))
    assert not fails, fails


@pytest.mark.parametrize("world", [2, 4])
def test_virtual_super_learner(world):
    """Every factorisation world = S*R, R learners co-located on one GPU: replicas
    bitwise equal, log replay bitwise for R <= 2 and within reading c11 for R = 4
    (the in-process sum runs in rank order)."""
    import mp_super
    fails = _virtual(world, lambda r, G: mp_super.body(r, world, 0, G))
    assert not fails, fails
