#!/bin/bash
# NVLink evidence on a G-GPU box: NVML calibration, ncu counters of the fused
# engine kernel (in-process, one-sided all-cross), and bench.py at N = G.
# usage: tools/gpurun_nvlink.sh G tag [skip_tests]
G=$1; T=$2
set -x
python -c "import __graft_entry__ as g; g.build()"
if [ "$3" != "skip_tests" ]; then
  timeout 900 python -m pytest tests/test_multigpu.py -v -k "$G" > gpurun_out/${T}_multigpu.log 2>&1
fi
timeout 120 python tools/nvml_nvlink_probe.py > gpurun_out/${T}_nvml_probe.json 2>&1
M=nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --devices 0 -k regex:k_engine -c 2 --metrics $M --clock-control none --csv \
  --log-file gpurun_out/${T}_ncu_inproc_G${G}.csv python tools/nvlink_ncu_inproc.py $G > gpurun_out/${T}_ncu_inproc_G${G}.log 2>&1
timeout 900 ncu --devices 0 -k regex:k_engine -s 1 -c 1 --set full --import-source on --clock-control none \
  -o gpurun_out/${T}_k_engine_allcross_G${G} python tools/nvlink_ncu_inproc.py $G > gpurun_out/${T}_ncu_full_G${G}.log 2>&1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus $G > gpurun_out/${T}_bench_N${G}.json 2> gpurun_out/${T}_bench_N${G}.err
