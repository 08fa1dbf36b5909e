for i in 1 2; do for v in prev main; do
  if [ $v = main ]; then L=paper_1710_06952_b200/libadpsgd.so; else L=build_ab/$v/libadpsgd.so; fi
  echo "== $v $(ADPSGD_LIB=$L timeout 300 python tools/config2_leg.py 2>&1 | tail -1)"
done; done
