# A/B of the engine tile size on the N=1 headline (bench --no-extras), twice each
for i in 1 2; do for v in main t1024 t768 t768s3 t512; do
  if [ $v = main ]; then L=paper_1710_06952_b200/libadpsgd.so; else L=build_ab/$v/libadpsgd.so; fi
  hb=$(ADPSGD_LIB=$L timeout 300 python bench.py --no-extras --steps 20 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), round(d['roofline']['frac'],4), round(d['e2e']['value']), d['clocks']['sm_mhz'])")
  echo "== $v headline $hb"
done; done
for v in t768; do
  ADPSGD_LIB=build_ab/$v/libadpsgd.so timeout 600 ncu -k regex:k_engine -s 1 -c 1 --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none python tools/prof_engine.py --updates 256 --runs 2 > gpurun_out/ab_${v}_ncu.log 2>&1
  grep -E "dram__bytes|gpu__time|lts__t_sectors|algorithmic" gpurun_out/ab_${v}_ncu.log | tail -8
done
