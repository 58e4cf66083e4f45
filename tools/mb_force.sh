# MBConv planner experiments: time (and check) forced TMEM / chunk plans
for f in "" "1,2,1,64" "1,2,2,32" "0,2,2,64" "1,1,2,32"; do
  echo "== force '$f'"
  WL_MB_FORCE="$f" python tools/prof_block.py mb14 2>&1 | tail -2
  WL_MB_FORCE="$f" python - <<'PY' 2>&1 | tail -2
import sys; sys.path.insert(0, ".")
import numpy as np
from oracle import model as om
from paper_2404_03617_b200.blocks import init_weights
from paper_2404_03617_b200.core import MBConv, TensorDims
from paper_2404_03617_b200.machine import build_schedule, execute_numeric
b, d = MBConv(8, 4, 0.25), TensorDims(2, 14, 14, 128)
rng = np.random.default_rng(0)
s = build_schedule(b, d)
w = {n: v.astype(np.float16).astype(np.float32) for n, v in init_weights(s, rng).items()}
x = rng.standard_normal((2, 14, 14, 128)).astype(np.float16).astype(np.float32)
got = execute_numeric(s, dict(w, x=x)); ref = om.unit_forward(b, w, x)
print("max_rel", np.abs(got - ref).max() / np.abs(ref).max())
PY
done
