"""Launch each hot kernel of the TGV / Poisson step twice on an ne^3 lx=8 box, for
ncu captures of the benched sizes (bench.py's roofline.traffic):

    ncu --set full --clock-control none -k regex:'mgs2|ax8t|dssum_blk' -c 14 \\
        -o gpurun_out/r2_ncu_<ne> python tools/kernel_probe.py <ne>

Kernels: the GMRES MGS pass (mgs2_kernel<1,1,0,0>), the pressure operator's Ax
with the fused Jacobi scaling (ax8t_kernel<0,0,1,0>), the masked Poisson Ax
(ax8t_kernel<0,1,0,0>), the plain Ax (ax8t_kernel<0,0,0,0>: the TGV pressure
operator bench.py times) and the element-blocked dssum (add and masked).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from bench import poisson_space
    from paper_2207_07098_b200 import _device, _lib
    from paper_2207_07098_b200.operators import GlobalOp

    ne = int(sys.argv[1]) if len(sys.argv) > 1 else 48
    dev = torch.device("cuda", 0)
    sp, mask, f = poisson_space(ne, dev)
    P = sp.n_points
    g = torch.Generator(device="cpu").manual_seed(1)
    u = torch.randn(sp.shape, generator=g, dtype=torch.float64).to(dev)
    pre = (torch.rand(sp.shape, generator=g, dtype=torch.float64) + 0.5).to(dev)
    w = torch.empty_like(u)
    opm = GlobalOp(sp, 1.0, 0.0, mask)
    op = GlobalOp(sp, 1.0, 0.0, None)
    vp, vn = torch.randn_like(u), torch.randn_like(u)
    h = torch.tensor([1e-9, 0.0], dtype=torch.float64, device=dev)
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    wk = _device.workspace(dev)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        _lib.call("sf_mgs_step_f64", _lib.ptr(w), _lib.ptr(vp), _lib.ptr(h), _lib.ptr(vn), None, None,
                  _lib.ptr(sp.gs.mult8), 0, P, *wk.args(), _lib.ptr(out), None, st)
        op.apply_into(u, w, pre=pre)          # ax8t<0,0,1,0> + dssum_blk<0>
        opm.apply_into(u, w)                  # ax8t<0,1,0,0> + dssum_blk<2>
        op.apply_into(u, w)                   # ax8t<0,0,0,0> + dssum_blk<0>
    torch.cuda.synchronize()
    print(f"kernel_probe ne={ne} P={P} ok")


if __name__ == "__main__":
    main()
