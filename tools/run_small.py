"""Tiny fwd+bwd launches of every kernel family and variant (for
compute-sanitizer runs): ranks 1-3, head_dim 16/32/64/128, fp16, bf16 (the
precise and the plain variant), fp32; the small-tile forward (3 CTAs/SM);
tensor-core and CUDA-core paths; contiguous and strided (heads-last) layouts."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import na_synth  # noqa: E402
import paper_2403_04690_b200 as na  # noqa: E402

cases = [
    ([300], [33], [2], [1], 64, torch.float16),
    ([20, 27], [7, 5], [2, 1], [0, 0], 32, torch.bfloat16),
    ([6, 10, 12], [3, 5, 5], [1, 1, 2], [1, 0, 0], 64, torch.float16),
    ([300], [33], [2], [1], 64, torch.bfloat16),
    ([20, 27], [7, 5], [2, 1], [0, 0], 64, torch.float16),
    ([6, 10, 12], [3, 5, 5], [1, 1, 2], [1, 0, 0], 32, torch.bfloat16),
    ([50], [7], [1], [0], 16, torch.float32),
    ([300], [33], [2], [1], 128, torch.float16),             # head_dim 128
    ([9, 20], [5, 7], [1, 2], [0, 1], 128, torch.bfloat16),
    ([6, 10, 12], [3, 5, 5], [1, 1, 2], [1, 0, 0], 128, torch.float16),
    ([56, 56], [7, 7], [8, 8], [0, 0], 32, torch.float16),   # small-tile forward (7x7 classes)
    ([24, 20], [5, 5], [1, 1], [0, 0], 16, torch.float16),
    ([40, 40], [13, 11], [1, 1], [0, 0], 64, torch.bfloat16),  # bf16 plain variant (143 keys)
]
for ext, ker, dil, cau, d, dt in cases:
    cfg = na_synth.small_config(ext, ker, dil, cau, head_dim=d, dtype=dt)
    q, k, v, do = na_synth.make_inputs(cfg, device="cuda", salt=2)
    kw = dict(kernel_size=ker, dilation=dil, is_causal=[bool(c) for c in cau])
    for impl in (["tc", "simt"] if dt != torch.float32 else ["simt"]):
        o, lse = na.na_fwd(q, k, v, impl=impl, **kw)
        na.na_bwd(q, k, v, o, do, lse, impl=impl, **kw)
# strided: heads-last [B, X, H, D] storage viewed as [B, H, X, D]; B = 2 with
# H = 2 does not merge (one launch set per batch entry)
for ext, ker, dt, impl in (([30, 12], [5, 3], torch.float16, "tc"), ([40], [7], torch.float32, "simt")):
    R = len(ext)
    cfg = na_synth.small_config(ext, ker, head_dim=32, batch=2, heads=2, dtype=dt)
    to_hl, from_hl = (0, *range(2, 2 + R), 1, 2 + R), (0, 1 + R, *range(1, 1 + R), 2 + R)
    q, k, v, do = (t.permute(to_hl).contiguous().cuda().permute(from_hl)
                   for t in na_synth.make_inputs(cfg, salt=2))
    o, lse = na.na_fwd(q, k, v, ker, impl=impl)
    na.na_bwd(q, k, v, o, do, lse, ker, impl=impl)
torch.cuda.synchronize()
print("ok")
