"""One cubics_propagate root fixpoint of gen_random(VARS, WIDTH, CONS, SEED) (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1909_09213_b200 import models  # noqa: E402
from paper_1909_09213_b200 import solver as S  # noqa: E402

v, w, c, s = (int(x) for x in sys.argv[1:5])
m = S.parse_model(models.gen_random(v, w, c, s))
for _ in range(int(sys.argv[5]) if len(sys.argv) > 5 else 1):
    d, fx = S.propagate_fixpoint(m)
print(fx)
