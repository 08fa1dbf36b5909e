# A/B of engine constants on the config-2 small-event legs and the N=1 headline (bench --no-extras)
for v in main t768 c2; do
  if [ $v = main ]; then L=paper_1710_06952_b200/libadpsgd.so; else L=build_ab/$v/libadpsgd.so; fi
  c2=$(ADPSGD_LIB=$L timeout 300 python tools/config2_leg.py 2>&1 | tail -1 | cut -c1-120)
  hb=$(ADPSGD_LIB=$L timeout 300 python bench.py --no-extras --steps 20 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), round(d['roofline']['frac'],4))")
  echo "== $v $c2 | headline $hb"
done
