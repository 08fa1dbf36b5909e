for i in 1 2; do
for lib in build_ab/old/libadpsgd.so paper_1710_06952_b200/libadpsgd.so; do
  echo "== $lib"; ADPSGD_LIB=$lib timeout 300 python tools/mlp_legs.py 2>&1 | head -2 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); d=d.get('mlp_config3',d); print(round(d['updates_per_s']))"
done; done
