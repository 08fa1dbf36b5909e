#!/bin/bash
# one-GPU evidence for the round: full -m gpu suite + smoke, the bench line, ncu launch
# list of the bench command, a full ncu capture of k_engine (bench configuration, 256-event
# launch) and of the MLP GEMMs.   usage: tools/gpurun_r02_final1.sh tag
T=$1
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/${T}_gputest.log 2>&1; echo rc=$? >> gpurun_out/${T}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --steps 3 --warmup 3 --no-extras > /dev/null 2>&1
timeout 600 ncu -k regex:k_engine -s 1 -c 1 --set full --import-source on --clock-control none \
  -o gpurun_out/${T}_k_engine_full python tools/prof_engine.py --updates 256 --runs 2 > gpurun_out/${T}_prof_engine.log 2>&1
timeout 600 ncu -k regex:k_gemm -s 2 -c 2 --set full --import-source on --clock-control none \
  -o gpurun_out/${T}_gemm_full python tools/prof_mlp.py > /dev/null 2>&1
# per-CTA phase trace of the GEMM kernels (tools/gemm_probe_build.sh builds build_probe/base/probe)
timeout 120 ./build_probe/base/probe > gpurun_out/${T}_gemm_phase_trace.txt 2>&1
timeout 300 python tools/mlp_host_bound.py > gpurun_out/${T}_mlp_host_bound.txt 2>&1
