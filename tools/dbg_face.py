import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2209_01877_b200 as P
from gpu_helpers import meshes, oracle_state
for order in (0, 1, 2):
    name, m = meshes()[0]
    gas = P.GasModel(); geo = P.compute_geometry(m, order)
    bcs = P.BoundaryConditions(P.freestream_conserved(gas, 0.4, 10.0))
    disc, c = oracle_state(m, order)
    try:
        buf = P.face_flux_pass(P.DofState(torch.from_numpy(c).cuda()), None, m, geo, bcs, gas)
        f = buf.inviscid.cpu().numpy(); ref = disc.flux_pass(c)
        print(order, 'ok', np.abs(f-ref).max())
    except Exception as e:
        print(order, 'ERR', e)
        from paper_2209_01877_b200.dg import _get_disc
        d = _get_disc(m, geo, gas, bcs)
        rows = d.to_reference(torch.from_numpy(c).cuda())
        d.reset_errors(); hb = d.face_flux(rows, 64)
        h = hb.cpu().numpy()[:4, :5*d.nqf]
        print(' H[0:4]', h)
        print(' ref', disc.flux_pass.__self__ if False else disc.rhs.__name__)
        print(' fcells', m.face_cells[:4], 'slots', m.face_slots[:4], 'info', geo.finfo[:4])
        print(' err', d.err.cpu().numpy().astype(np.uint32))
