# N=4 A/B of ADPSGD_CROSS_DIV (default build = 4 vs build_ab/x1), then the GPU suite
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29800
for v in default x1 default x1; do
  if [ $v = default ]; then L=""; else L="ADPSGD_LIB=build_ab/$v/libadpsgd.so"; fi
  P=$((P+1)); env $L timeout 300 $TR --master-port $P bench.py --gpus 4 --no-extras 2>/dev/null | grep '^{' | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$v', round(j['value']), round(j['roofline']['frac'],3))"
  P=$((P+1)); env $L timeout 300 $TR --master-port $P tools/ab_nvlink.py --mode run --wpg 32 --variants 0 --events 1024 --placement xor 2>&1 | grep -i "GB/s" | tail -1
done
timeout 1300 python -m pytest tests -m gpu -q 2>&1 | tail -3
