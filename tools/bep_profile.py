"""One fused BEP column chunk at cfg4 (for ncu launch lists): python tools/bep_profile.py [ncols]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from dpm_inputs import get_config  # noqa: E402
from paper_1811_03557_b200 import api  # noqa: E402

nc = int(sys.argv[1]) if len(sys.argv) > 1 else 64
c = api.DPM.from_config(get_config("cfg4"))
c.bep_columns(0, nc)
torch.cuda.synchronize()
c.bep_columns(0, nc)
torch.cuda.synchronize()
print("ok")
