timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_gpu_parity.py -q -x -k "gemm or mlp or config3" 2>&1 | tail -1
timeout 300 python tools/mlp_legs.py 2>&1 | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read())
print(round(d['mlp_config3']['updates_per_s']), round(d['mlp_config3_free_running_1gpu']['updates_per_s']))
print([(x['M_batch'], x['bn'], x['splits'], round(x['us'],1), round(x['frac_tf32_peak'],3)) for x in d['mlp_gemm_sweep']['rows']])"
timeout 60 ./build_probe/base/probe | grep -A3 "GEMM1 bn 64 splits 16\|GEMM2\|^K/K\|^MN\|^K tma" | grep -v "setup\|start"
