# robustness: the -m gpu suite twice in a row and the opt-in 8-rank parity test three times
for i in 1 2; do timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/flaky_suite_$i.log 2>&1; echo "suite $i: $(tail -1 gpurun_out/flaky_suite_$i.log)"; done
for i in 1 2 3; do ADPSGD_TEST_WORLD8=1 timeout 400 python -m pytest tests/test_virtual_ranks.py -q -x -k world8 > gpurun_out/flaky_w8_$i.log 2>&1; echo "world8 $i: $(tail -1 gpurun_out/flaky_w8_$i.log)"; done
