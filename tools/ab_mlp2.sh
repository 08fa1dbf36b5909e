# A/B of the MLP GEMM variants (tools/ab_build.py builds build_ab/<v>)
for i in 1 2; do
for v in main one two; do
  if [ $v = main ]; then L=paper_1710_06952_b200/libadpsgd.so; else L=build_ab/$v/libadpsgd.so; fi
  echo "== $v $(ADPSGD_LIB=$L timeout 300 python tools/mlp_legs.py 2>&1 | head -2 | python -c "
import sys,json
out=[]
for l in sys.stdin:
    d=json.loads(l); d=d.get('mlp_config3',d); out.append(str(round(d['updates_per_s'])))
print(' '.join(out))")"
done; done
ADPSGD_LIB=build_ab/two/libadpsgd.so timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_gpu_parity.py -q -x -k "gemm or mlp or config3" 2>&1 | tail -1
