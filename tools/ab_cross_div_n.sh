# A/B of engine build variants (build_ab/<v>/libadpsgd.so; "default" = in-tree) at N=2 and N=4
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
P=29850
for rep in 1 2; do
for v in default x3 x6 gf; do
  if [ $v = default ]; then L=""; else L="ADPSGD_LIB=build_ab/$v/libadpsgd.so"; fi
  for N in 2 4; do
    P=$((P+1)); env $L timeout 300 $TR --nproc-per-node $N --master-port $P bench.py --gpus $N --no-extras 2>/dev/null | grep '^{' | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$v N=$N', round(j['value']), round(j['roofline']['frac'],3))"
  done
done
done
