import sys, torch
sys.path.insert(0, ".")
from paper_1704_08364_b200 import fourier_bp as F, phantom
from paper_1704_08364_b200.preprocess import center_beta
N=2048; k=64
plan=F.BstPlan(N,N)
vol=phantom.ellipsoid_volume(k, N, N, device="cuda"); vol += 0.01*torch.rand(vol.shape, device="cuda")
nat=F.native_plan(plan, F.FilterPlan(), False, 0)
ws=nat.new_workspace(31); out=torch.empty((k,N,N),device="cuda")
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    best=1e9
    for _ in range(reps):
        a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); best=min(best,a.elapsed_time(b))
    return best/k
bc=center_beta(vol,k,N,N,False,"auto")
sh,st=nat.pre_params(vol,k,bc,9)
print("center_beta", t(lambda: center_beta(vol,k,N,N,False,"auto")))
print("pre_params", t(lambda: nat.pre_params(vol,k,bc,9)))
print("run", t(lambda: nat.run("fbp", vol, out, k, 31, ws)))
print("run_pre", t(lambda: nat.run_pre(vol, out, k, 31, ws, sh, st)))
print("run_pre_noring", t(lambda: nat.run_pre(vol, out, k, 31, ws, sh, None)))
print("fbp_volume fused", t(lambda: F.fbp_volume(vol, plan, center="auto", rings=9, out=out, batch=31, check=False)))
print("fbp_volume plain", t(lambda: F.fbp_volume(vol, plan, out=out, batch=31, check=False)))
