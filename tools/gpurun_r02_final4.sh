#!/bin/bash
# 4-GPU evidence: multi-GPU parity (processes), ncu NVLink counters (G=2, 4), bench N=2 and N=4
T=$1
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_multigpu.py -v > gpurun_out/${T}_multigpu.log 2>&1
M=nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for G in 2 4; do
  timeout 600 ncu --devices 0 -k regex:k_engine -c 2 --metrics $M --clock-control none --csv \
    --log-file gpurun_out/${T}_ncu_inproc_G${G}.csv python tools/nvlink_ncu_inproc.py $G > gpurun_out/${T}_ncu_inproc_G${G}.log 2>&1
done
for N in 2 4; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29511 + N)) bench.py --gpus $N > gpurun_out/${T}_bench_N${N}.json 2> gpurun_out/${T}_bench_N${N}.err
done
