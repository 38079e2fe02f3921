"""The reference's own call with its own types: fused_layer_attention on
float32 NumPy [B, H, N, d] arrays, NumPy float32 result (attention.py:186-212),
timed at a production layout, after one warm-up call.

    python scripts/time_numpy_api.py [hunyuan|cogvideo|wan]"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2506_03065_b200 as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "hunyuan"
cfg = bench.CONFIGS[name]
layout = S.TokenLayout(*cfg["layout"])
H, d, n = cfg["heads"], cfg["d"], layout.total_tokens
rng = np.random.default_rng(0)
q, k, v = (rng.standard_normal((1, H, n, d), dtype=np.float32) for _ in range(3))
groups = S.group_heads(bench.assignment_for(cfg, S), S.block_grid(layout))
S.fused_layer_attention(q, k, v, groups)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    out = S.fused_layer_attention(q, k, v, groups)
    ts.append(round((time.perf_counter() - t0) * 1e3, 1))
print(json.dumps({"config": name, "numpy_fp32_call_ms": ts, "out_dtype": str(out.dtype),
                  "bytes_in": 3 * q.nbytes, "bytes_out": out.nbytes}))
