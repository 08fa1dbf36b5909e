"""Driver for an ncu capture of the tcgen05 3xTF32 GEMM: GEMM1 of the config-3 MLP
(X_b W1^T, 128 x 512 x 3072) and the same GEMM at M = 4096 (gemm_sweep's best
configurations).  Each call = 2 warm-up launches + 1 timed launch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_06952_b200 as P

for (m, n, k, splits) in ((128, 512, 3072, 8), (4096, 512, 3072, 1)):
    ms = P.gemm_tf32x3_bench(m, n, k, splits, 128, 1)
    print(f"M={m} N={n} K={k} splits={splits}: {ms * 1e3:.1f} us", flush=True)
