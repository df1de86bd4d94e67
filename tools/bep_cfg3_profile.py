"""cfg3 BEP columns (K = 242, n = 64) twice, for ncu launch lists of the Step-4b rebuild at small n."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from dpm_inputs import get_config  # noqa: E402
from paper_1811_03557_b200 import api  # noqa: E402

c = api.DPM.from_config(get_config(sys.argv[1] if len(sys.argv) > 1 else "cfg3"))
c.bep_columns(0, c.K)
torch.cuda.synchronize()
c.bep_columns(0, c.K)
torch.cuda.synchronize()
print("ok")
