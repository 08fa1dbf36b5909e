#!/bin/bash
# Multi-GPU evidence on a G-GPU box: multi-GPU parity tests, ncu NVLink counters
# of the fused engine kernel (in-process ranks, one-sided all-cross), and
# bench.py at N = 2 .. G.   usage: tools/gpurun_nvlink.sh G tag [skip_tests]
G=$1; T=$2
set -x
python -c "import __graft_entry__ as g; g.build()"
if [ "$3" != "skip_tests" ]; then
  timeout 900 python -m pytest tests/test_multigpu.py -v > gpurun_out/${T}_multigpu.log 2>&1
fi
M=nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --devices 0 -k regex:k_engine -c 2 --metrics $M --clock-control none --csv \
  --log-file gpurun_out/${T}_ncu_inproc_G${G}.csv python tools/nvlink_ncu_inproc.py $G > gpurun_out/${T}_ncu_inproc_G${G}.log 2>&1
for N in $(seq 2 $G); do
  if [ $N -eq 3 ]; then continue; fi
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29511 + N)) bench.py --gpus $N > gpurun_out/${T}_bench_N${N}.json 2> gpurun_out/${T}_bench_N${N}.err
done
