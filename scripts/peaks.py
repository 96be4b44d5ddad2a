"""Measure the FP64 roofline denominators on this GPU (csrc/pbad_peak.cu):
DFMA rate and dependent latency, DMMA (FP64 tensor core) rate.
    python scripts/peaks.py [out.json]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

res = {}
for rep in range(3):
    dfma, lat = bench.measured_fp64_peak(0)
    dmma = bench.measured_dmma_peak(0)
    res.setdefault("dfma_tflops", []).append(dfma)
    res.setdefault("dfma_latency_cycles", []).append(lat)
    res.setdefault("dmma_tflops", []).append(dmma)
res["note"] = ("k_dfma_peak: 8 independent DFMA chains per thread, 148 x 8 blocks of 256 threads; "
               "k_dmma_peak: 8 independent mma.sync.m8n8k4.f64 accumulators per warp (256 FMA each), "
               "same grid; best of 5 launches each, FMA = 2 FLOPs")
print(json.dumps(res, indent=1))
if len(sys.argv) > 1:
    json.dump(res, open(sys.argv[1], "w"), indent=1)
