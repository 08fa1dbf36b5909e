timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_gpu_parity.py -q -x -k "gemm or mlp or config3" > gpurun_out/r02zr_test.log 2>&1; tail -3 gpurun_out/r02zr_test.log
timeout 300 python tools/mlp_legs.py > gpurun_out/r02zr_mlp.json 2>&1; tail -c 3000 gpurun_out/r02zr_mlp.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02zr_mlp_launches.csv python tools/prof_mlp.py > /dev/null 2>&1
