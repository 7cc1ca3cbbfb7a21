#!/bin/bash
# runs the TMA probe over map locations x extras (prefetch / proxy fence / .shared::cta .tile), one process each
cd "$(dirname "$0")"
for w in 0 1; do for x in 0 1 2 3 4 7; do
  echo "== where=$w xtra=$x"; TMA_WHERE=$w TMA_X=$x ./tma2d_probe 2>&1 | tail -1
done; done
python - <<'PY'
import torch
a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
print("matmul ok", float((a @ a).float().abs().sum()))
PY
ncu --metrics gpu__time_duration.sum python -c "
import torch
a = torch.randn(4096, 4096, device='cuda', dtype=torch.bfloat16)
b = a @ a
torch.cuda.synchronize()" 2>&1 | grep -E "^\s+[a-zA-Z_].*\(" | head -5
