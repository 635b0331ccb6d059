import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from golden_util import load_case, oracle_plan, rel_l2
from oracle import bst_oracle as O
from paper_1704_08364_b200 import fourier_bp as F
c = load_case("shepp256"); op = oracle_plan(c)
plan = F.BstPlan(256, 256); nat = F.native_plan(plan, F.FilterPlan(), False, 0)
sino = torch.from_numpy(c["sino"]).cuda(); img = torch.empty((256, 256), device="cuda")
ws = nat.new_workspace(1); nat.reset_status(ws); nat.run("fbp", sino, img, 1, 1, ws); nat.read_status(ws)
lay = nat.layout(1); H = 256
pol = ws[lay["polar"]: lay["polar"] + 256 * H * 8].view(torch.float32).cpu().numpy().view(np.complex64).reshape(256, H)
h = O.ramp_filter(c["sino"].astype(np.float64), op)
Ahat, a, colsum = O.k1_polar(h, op)
err = np.abs(pol - Ahat)
print("row err max", np.argsort(-err.max(1))[:10], err.max(1)[np.argsort(-err.max(1))[:10]])
print("col err max", np.argsort(-err.max(0))[:10], err.max(0)[np.argsort(-err.max(0))[:10]])
print(pol[5, 60:66]); print(Ahat[5, 60:66])
