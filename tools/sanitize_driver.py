"""Small workloads for compute-sanitizer (tools/sanitize.sh): every kernel of
the library at L = 256 / 512 with batch 3 on two lanes (3 launch groups:
lane-1 workspace regions, texture views and the shared status word), the
host slab pipeline, the counts / frames / ss / ramp / forward / preprocess
entry points, the fused centre / ring load, full turn and nearest
interpolation (K2_TEXF / K2_TEXN over three launch groups)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1704_08364_b200 import fourier_bp as F  # noqa: E402
from paper_1704_08364_b200 import phantom, projector  # noqa: E402
from paper_1704_08364_b200.preprocess import FlatDarkFrames, preprocess_volume  # noqa: E402
from paper_1704_08364_b200.slices import AngleAxis, DetectorAxis, ImageGrid, Sinogram  # noqa: E402

torch.cuda.set_device(0)
for n in (128, 256):
    plan = F.BstPlan(n, n)
    vol = phantom.ellipsoid_volume(7, n, n, device="cuda")
    vol += 0.01 * torch.randn(vol.shape, device="cuda")
    a = F.fbp_volume(vol, plan, batch=3)                         # 3 groups on 2 lanes
    b = F.fbp_volume(vol.cpu(), plan, batch=3, chunk=4)          # host pipeline
    assert torch.equal(a.cpu(), b)
    F.fbp_volume(vol, plan, batch=3, kernel="none", scale=0.5)   # tb_bst_scaled
    F.fbp_volume(vol[:3].contiguous(), plan, batch=3, kernel="ss")
    frames = FlatDarkFrames(np.full((n, n), 2.0), np.zeros((n, n)))
    F.fbp_volume(torch.exp(-vol) * 2.0, plan, batch=3, frames=frames)  # fused normalisation (constant frames)
    fr2 = FlatDarkFrames(np.full((n, n), 2.0) + np.linspace(0, 0.1, n)[None, :], np.full((n, n), 0.01))
    F.fbp_volume(torch.exp(-vol) * 2.0, plan, batch=3, frames=fr2)     # per-sample frames table
    preprocess_volume(vol, plan, center=0.5, rings=9)
    F.fbp_volume(vol, plan, batch=3, center=0.5, rings=9)     # centre / rings fused into K1 (tb_fbp_pre)
    F.fbp_volume(vol, plan, batch=3, center=-1.25)             # centring only (no stripe profile)
    F.fbp_volume(vol, F.BstPlan(n, n, interp="nearest"), batch=3)                  # K2_TEXN, 3 groups
    F.fbp_volume(torch.cat([vol, vol.flip(2)], dim=1).contiguous(), plan, batch=3,
                 full_turn=True)                                                  # K2_TEXF, 3 groups
    y = Sinogram(DetectorAxis(n), AngleAxis(n), vol[3].cpu().numpy().astype(np.float64))
    F.ramp_filter(y)
    F.fbp(y, F.BstPlan(n, n, output_n=n // 2 + 1))               # Nyquist lines, non-crop-half K2/K3
    F.fbp(y, F.BstPlan(n, n, interp="nearest"))                  # K2_TEXN (single slice)
    yf = Sinogram(DetectorAxis(n), AngleAxis(2 * n, full_turn=True),
                  np.vstack([y.data, y.data[:, ::-1]]))
    F.fbp(yf, F.BstPlan(n, n))                                   # full-turn K2_TEXF
    projector.forward_project(ImageGrid(n, a[0].cpu().numpy().astype(np.float64)), DetectorAxis(n), AngleAxis(n))
torch.cuda.synchronize()
print("sanitize_driver ok")
