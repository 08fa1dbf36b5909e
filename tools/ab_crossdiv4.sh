for N in 2 4; do
for v in main d2 d8 main d2 d8; do
  if [ $v = main ]; then L=paper_1710_06952_b200/libadpsgd.so; else L=build_ab/$v/libadpsgd.so; fi
  ADPSGD_LIB=$L timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + N)) bench.py --gpus $N --no-extras --steps 20 > gpurun_out/r02zd_${v}_$N.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/r02zd_${v}_$N.json').read().strip().splitlines()[-1]); print('N=$N', '$v', round(d['value']), round(d['updates_per_s']), round(d['roofline']['frac'],4))" >> gpurun_out/r02zd_summary.txt
done; done
