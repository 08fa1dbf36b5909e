"""tcgen05 3xTF32 GEMM utilisation at the config-3 MLP shapes, M in {128, 1024, 4096}
(SURVEY 8(d)): GEMM1 Z1 = X_b W1^T (M x 512 x 3072) and GEMM2 dW1 = dZ1^T X_b
(512 x 3072 x M).  3xTF32 issues three TF32 MMAs per product, so tensor work =
3 x 2MNK; the TF32 dense peak is taken as half the measured bf16 peak."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_06952_b200 as P


def sweep(reps=20):
    try:
        pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                         "MEASURED_PEAKS.json")))
        tf32_peak = pk["bf16_tflops"] / 2.0
        src = "MEASURED_PEAKS.json bf16_tflops / 2 (nominal TF32:BF16 ratio)"
    except Exception:
        tf32_peak, src = 1125.0, "nominal 2.25 PF bf16 / 2"
    rows = []
    for M in (128, 1024, 4096):
        for name, (m, n, k) in (("gemm1 X_b.W1^T", (M, 512, 3072)), ("gemm2 dZ1^T.X_b", (512, 3072, M))):
            best = None
            for bn in (64, 128):
                for splits in (1, 2, 4, 8, 16):
                    if k % (32 * splits) or n % bn:
                        continue
                    ms = P.gemm_tf32x3_bench(m, n, k, splits, bn, reps)
                    if best is None or ms < best[0]:
                        best = (ms, bn, splits)
            ms, bn, splits = best
            flop = 2.0 * m * n * k
            rows.append({"gemm": name, "M_batch": M, "shape_MNK": [m, n, k], "bn": bn, "splits": splits,
                         "us": ms * 1e3, "tflops_fp32_equiv": flop / (ms / 1e3) / 1e12,
                         "tensor_tflops_tf32": 3 * flop / (ms / 1e3) / 1e12,
                         "frac_tf32_peak": 3 * flop / (ms / 1e3) / 1e12 / tf32_peak})
    return {"tf32_peak_tflops": tf32_peak, "peak_source": src, "rows": rows}


if __name__ == "__main__":
    out = sweep()
    print(f"TF32 peak {out['tf32_peak_tflops']:.0f} TFLOP/s ({out['peak_source']})")
    for r in out["rows"]:
        print(f"{r['gemm']:18s} M={r['M_batch']:5d} {str(r['shape_MNK']):20s} bn={r['bn']} splits={r['splits']} "
              f"{r['us']:8.1f} us  {r['tflops_fp32_equiv']:6.1f} TF/s fp32-eq  {r['tensor_tflops_tf32']:6.1f} "
              f"TF/s tensor  {r['frac_tf32_peak']:.3f} of TF32 peak")
