# A/B: previous commit (build_ab/prev) vs the working tree, config-3 replay / free-running / host-bound
for i in 1 2; do
for v in prev main; do
  if [ $v = main ]; then L=paper_1710_06952_b200/libadpsgd.so; else L=build_ab/$v/libadpsgd.so; fi
  echo "== $v $(ADPSGD_LIB=$L timeout 300 python tools/mlp_legs.py 2>&1 | head -2 | python -c "
import sys,json
out=[]
for l in sys.stdin:
    d=json.loads(l); d=d.get('mlp_config3',d); out.append(str(round(d['updates_per_s'])))
print(' '.join(out))")"
done; done
timeout 200 python tools/mlp_host_bound.py
