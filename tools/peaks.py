"""Measured compute peaks of this B200 beside MEASURED_PEAKS.json:
FP32 FFMA (SIMT) and FP32-accurate 3xTF32 mma.sync.  usage: python tools/peaks.py [out.json]"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_02234_b200._lib import check, lib

import torch

L = lib()
f32, tc = ctypes.c_double(), ctypes.c_double()
best32 = best_tc = 0.0
for _ in range(3):
    check(L.hmdp_peak_fp32(0, 300, ctypes.byref(f32)))
    check(L.hmdp_peak_tf32x3(0, 300, ctypes.byref(tc)))
    best32, best_tc = max(best32, f32.value), max(best_tc, tc.value)
res = {"gpu": torch.cuda.get_device_name(0),
       "fp32_ffma_tflops": best32,
       "tf32x3_mma_sync_tflops": best_tc,
       "tf32_mma_sync_raw_tflops": 3 * best_tc,
       "how": "hmdp_peak_fp32 / hmdp_peak_tf32x3 (csrc/hmdp_probe.cu), best of 3, CUDA events; "
              "3xTF32 counts each hi/lo triple of m16n8k8 MMAs as one product"}
print(json.dumps(res))
if len(sys.argv) > 1:
    json.dump(res, open(sys.argv[1], "w"), indent=1)
