"""BEP factorisation at cfg4 (for ncu launch lists): python tools/factor_profile.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from dpm_inputs import get_config  # noqa: E402
from paper_1811_03557_b200 import api  # noqa: E402

c = api.DPM.from_config(get_config("cfg4"))
PgE, B = c.bep_columns(0, c.K)
c.bep_factor(B)
torch.cuda.synchronize()
c.bep_factor(B)
torch.cuda.synchronize()
print("ok")
