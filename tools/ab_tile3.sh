# valid tile sizes (multiples of 512) x stages on the N=1 headline, twice each
for i in 1 2; do for v in main t1024s3 t512s4; do
  if [ $v = main ]; then L=paper_1710_06952_b200/libadpsgd.so; else L=build_ab/$v/libadpsgd.so; fi
  hb=$(ADPSGD_LIB=$L timeout 300 python bench.py --no-extras --steps 20 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])")
  echo "== $v headline $hb"
done; done
