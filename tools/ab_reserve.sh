# A/B: cross events on a reserved CTA range (build_ab/rsv, -DADPSGD_CROSS_RESERVE=1) vs default
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P=29870
for rep in 1 2; do
for v in default rsv; do
  if [ $v = default ]; then L=""; else L="ADPSGD_LIB=build_ab/$v/libadpsgd.so"; fi
  for N in 2 4; do
    P=$((P+1)); env $L timeout 300 $TR --nproc-per-node $N --master-port $P bench.py --gpus $N --no-extras 2>/dev/null | grep '^{' | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$v N=$N', round(j['value']), round(j['roofline']['frac'],3))"
  done
done
done
P=$((P+1)); ADPSGD_LIB=build_ab/rsv/libadpsgd.so timeout 300 $TR --nproc-per-node 2 --master-port $P tools/engine_breakdown.py 2>/dev/null
P=$((P+1)); ADPSGD_LIB=build_ab/rsv/libadpsgd.so timeout 400 $TR --nproc-per-node 2 --master-port $P tests/mp_worker.py 2>&1 | grep MULTIGPU
P=$((P+1)); ADPSGD_LIB=build_ab/rsv/libadpsgd.so timeout 300 $TR --nproc-per-node 4 --master-port $P tools/ab_nvlink.py --mode run --wpg 32 --variants 0 --events 1024 --placement xor 2>&1 | grep "GB/s" | tail -1
