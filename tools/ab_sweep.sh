for v in main two; do
  if [ $v = main ]; then L=paper_1710_06952_b200/libadpsgd.so; else L=build_ab/$v/libadpsgd.so; fi
  ADPSGD_LIB=$L timeout 300 python -c "
import sys; sys.path.insert(0,'tools'); sys.path.insert(0,'.')
import gemm_sweep
r=gemm_sweep.sweep(reps=10)
print('$v', [(x['M_batch'], x['bn'], x['splits'], round(x['us'],1), round(x['frac_tf32_peak'],3)) for x in r['rows']])"
done
