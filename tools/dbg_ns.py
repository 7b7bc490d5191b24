"""Diagnostics: GPU 2D viscous passes vs the oracle, bit for bit (FP32)."""
import sys

import numpy as np
import torch

sys.path.insert(0, "tests")
from conftest import golden_path  # noqa: E402
from oracle import mesh as OM  # noqa: E402
from oracle import solver as S  # noqa: E402
from paper_2209_01877_b200 import twod  # noqa: E402

cfg = dict(gen_kind="quad", gen_nx=96, gen_ny=4, gen_extent=(0.0, 0.0, 12.0, 0.5), initial_kind="pulse",
           initial_x0=6.0, initial_y0=0.25, pulse_amplitude=0.2, pulse_sigma=0.3, mach=0.4, order=1, cfl=0.5,
           ivis=1, mu_dyn=0.002, max_iterations=120, precision_mode="mp_fixed", switch_iter=70)
_, hist, m, t = twod.run2d(twod.RunConfig2D(log_every=1, **cfg))
ref = np.array([[float(x) for x in r.split(",")[1:5]] for r in open(golden_path("residuals_ns_mp.csv")).read().split()[1:]])
got = np.array(hist.res)
rel = np.abs(got - ref) / np.abs(ref)
for i in (0, 1, 2, 5, 10, 30, 60, 69, 70, 71, 90, 119):
    print(i, rel[i])
# single-pass comparison at f32 on the initial state
om = OM.quad_grid(96, 4, (0.0, 0.0, 12.0, 0.5))
gas = S.Gas(mu=0.002, ivis=1)
spec = S.RunSpec(mesh=om, gas=gas, order=1, initial="pulse", x0=6.0, y0=0.25, amplitude=0.2, sigma=0.3, mach=0.4)
disc = S.make_disc(om, 1, gas, 0.4, 0.0)
c = S.initial_state(spec, disc).astype(np.float32)
_, qinf = twod.freestream_2d(1.4, 1.0, 0.4, 0.0)
dev = twod.Device2D(m, t, 1.4, qinf, mu=0.002, ivis=1)
u = torch.from_numpy(np.ascontiguousarray(c)).cuda()
aux_g = dev.aux_gradient(u).cpu().numpy()
aux_o = disc.aux_gradient(np.ascontiguousarray(c))
print("aux f32 identical:", np.array_equal(aux_g, aux_o), "n diff", np.sum(aux_g != aux_o), "of", aux_g.size)
fi, fv, fq = (x.cpu().numpy() for x in dev.face_flux_ns(u, torch.from_numpy(aux_o).cuda()))
oi, ov, oq = disc.flux_pass_ns(np.ascontiguousarray(c), aux_o)
for nm, a, b in (("finv", fi, oi), ("fvis", fv, ov), ("fqhat", fq, oq)):
    d = a != b
    print(nm, "n diff", int(d.sum()), "of", a.size, "faces", np.unique(np.nonzero(d)[0])[:20])
bc = m.boundary_kind_codes()
print("boundary faces", np.nonzero(bc > 0)[0][:10])
r_g = dev.accumulate_ns(u, torch.from_numpy(aux_o).cuda(), torch.from_numpy(oi).cuda(), torch.from_numpy(ov).cuda()).cpu().numpy()
r_o = disc.rhs_pass_ns(np.ascontiguousarray(c), aux_o, oi, ov)
print("rhs n diff", int((r_g != r_o).sum()), "of", r_g.size)

# lockstep: oracle vs GPU RK2 steps at FP32, first divergence
uo = np.ascontiguousarray(c)
ug = torch.from_numpy(uo.copy()).cuda()


def cmp_passes(x, tag):
    xa = np.ascontiguousarray(x)
    xg = torch.from_numpy(xa.copy()).cuda()
    ao = disc.aux_gradient(xa)
    ag = dev.aux_gradient(xg).cpu().numpy()
    fo = disc.flux_pass_ns(xa, ao)
    fg = [t_.cpu().numpy() for t_ in dev.face_flux_ns(xg, torch.from_numpy(ao).cuda())]
    ro = disc.rhs_pass_ns(xa, ao, fo[0], fo[1])
    rg = dev.accumulate_ns(xg, torch.from_numpy(ao).cuda(), torch.from_numpy(fo[0]).cuda(),
                           torch.from_numpy(fo[1]).cuda()).cpu().numpy()
    dto = S.local_dt_field(disc, xa, 0.5, 1)
    dtg = dev.local_dt(xg, 0.5, 1).cpu().numpy()
    bad = {"aux": np.nonzero((ao != ag).reshape(ao.shape[0], -1).any(1))[0],
           "finv": np.nonzero((fo[0] != fg[0]).reshape(fo[0].shape[0], -1).any(1))[0],
           "fvis": np.nonzero((fo[1] != fg[1]).reshape(fo[1].shape[0], -1).any(1))[0],
           "rhs": np.nonzero((ro != rg).reshape(ro.shape[0], -1).any(1))[0],
           "dt": np.nonzero(dto != dtg)[0]}
    print(tag, {k: v[:8].tolist() for k, v in bad.items() if v.size})
    for f in bad["finv"][:2]:
        print(" face", f, "bc", bc[f], "cells", m.face_cells[f], "normal", m.face_normal[f])
        print("  fqhat o", fo[2][f].tolist())
        print("  fqhat g", fg[2][f].tolist())
        print("  finv o", fo[0][f].tolist())
        print("  finv g", fg[0][f].tolist())
        iL = m.face_cells[f][0]
        np.save("gpurun_out/dbg_face.npy", np.concatenate([xa[iL].ravel().astype(np.float64),
                                                          fo[2][f].ravel().astype(np.float64)]))
    return bad


for it in range(30):
    dto = S.local_dt_field(disc, uo, 0.5, 1)
    n = uo.shape[0]
    # stage by stage
    L = S._clib.lib()
    r0o = disc.rhs(uo)
    u1o = np.empty_like(uo)
    L.ora_axpy_f32(n, 4 * 3, S._clib.ptr(uo), S._clib.ptr(r0o), S._clib.ptr(dto), S._clib.ptr(u1o))
    ug_new, _ = dev.rk2_step(ug, torch.from_numpy(dto).cuda())
    uo_new = S.rk2_step(uo, dto, disc.rhs)
    if not np.array_equal(uo_new, ug_new.cpu().numpy()):
        print("first divergence in step", it)
        cmp_passes(uo, "stage0")
        cmp_passes(u1o, "stage1")
        break
    uo, ug = np.ascontiguousarray(uo_new), ug_new
