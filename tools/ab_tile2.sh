# A/B of engine tile size / stages on the N=1 headline (bench --no-extras), twice each
for i in 1 2; do for v in main t768s3 t768s4 t640s3 t896s3 t1152s3 t1536s3; do
  if [ $v = main ]; then L=paper_1710_06952_b200/libadpsgd.so; else L=build_ab/$v/libadpsgd.so; fi
  hb=$(ADPSGD_LIB=$L timeout 300 python bench.py --no-extras --steps 20 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), round(d['roofline']['frac'],4), round(d['e2e']['value']), d['clocks']['sm_mhz'])")
  echo "== $v headline $hb"
done; done
