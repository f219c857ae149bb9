"""Check dkss_kernel_launches(): direct launches (profile path) and graph replays (device path)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1503_04955_b200._native import kernel_launches
from paper_1503_04955_b200.dkss import device_plan
from paper_1503_04955_b200.plan import dkss_select_params
from paper_1503_04955_b200.words import int_to_u32

pl = dkss_select_params(1 << 20)
dp = device_plan(pl, 0)
nl, npl = dp.info["operand_limbs"], dp.info["product_limbs"]
A = torch.from_numpy(int_to_u32(12345, nl).view(np.int32)).cuda()
C = torch.zeros(npl, dtype=torch.int32, device="cuda")
n0 = kernel_launches()
prof = dp.profile_device(1, A.data_ptr(), A.data_ptr(), nl, C.data_ptr(), 0)
n1 = kernel_launches()
for _ in range(3):
    dp.mul_device(1, A.data_ptr(), A.data_ptr(), nl, C.data_ptr(), npl, 0)
torch.cuda.synchronize()
n2 = kernel_launches()
print("profile launches", len(prof), "counted", n1 - n0, "| 3 graph replays counted", n2 - n1, "info", dp.info)
