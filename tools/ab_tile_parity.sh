# parity of the engine variants: every engine / free-running test, plus the smoke
for v in t768 t896s3; do
  echo "== $v: $(ADPSGD_LIB=build_ab/$v/libadpsgd.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_appa_gpu.py tests/test_virtual_ranks.py -q -x 2>&1 | tail -1)"
  ADPSGD_LIB=build_ab/$v/libadpsgd.so timeout 600 ncu -k regex:k_engine -s 1 -c 1 --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_op_write.sum --clock-control none python tools/prof_engine.py --updates 256 --runs 2 > gpurun_out/ab_${v}_ncu2.log 2>&1
  grep -E "dram__bytes|gpu__time|lts__t_sectors|algorithmic" gpurun_out/ab_${v}_ncu2.log | tail -8
done
timeout 600 ncu -k regex:k_engine -s 1 -c 1 --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_op_write.sum --clock-control none python tools/prof_engine.py --updates 256 --runs 2 > gpurun_out/ab_main_ncu2.log 2>&1
grep -E "dram__bytes|gpu__time|lts__t_sectors|algorithmic" gpurun_out/ab_main_ncu2.log | tail -8
