set -x
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
P=29700
for v in default x2 x4 x8; do
  if [ $v = default ]; then L=""; else L="ADPSGD_LIB=build_ab/$v/libadpsgd.so"; fi
  for c in 0 -1; do
    P=$((P+1)); env $L timeout 300 $TR --master-port $P bench.py --gpus 2 --no-extras --coop=$c 2>/dev/null | grep '^{' | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$v coop=$c', round(j['value']), round(j['roofline']['frac'],3), round(j['nvlink']['per_gpu_per_direction_gbs'],1))"
  done
  P=$((P+1)); env $L timeout 300 $TR --master-port $P tools/ab_nvlink.py --mode run --wpg 32 --variants 0 --events 512 2>&1 | grep -i "gb/s\|GB" | tail -2
done
P=$((P+1)); ADPSGD_LIB=build_ab/x4/libadpsgd.so timeout 400 $TR --master-port $P tests/mp_worker.py 2>&1 | grep MULTIGPU
