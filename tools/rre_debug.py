import sys, numpy as np, torch
sys.path.insert(0, ".")
import oracle as orc
from paper_2301_01718_b200 import inputs
from paper_2301_01718_b200 import hrom as H
wl = inputs.config(2, steps=inputs.config(2).w + 6, delta=0.99)
q0 = inputs.initial_condition(wl)
rom = H.HybridROM(wl); rom.set_state(torch.from_numpy(q0).cuda())
R = orc.Run(wl, q0)
for k in range(1, wl.w):
    rom.step(); R.step()
eg = rom.indicator().cpu().numpy(); eo = R.eps()
mg = H.cells_from_mask(wl, rom.mask()); mo = R.mask()
print("k", k, "sizes", mg.sum(), mo.sum(), "diff cells", np.nonzero(mg != mo)[0][:10])
m2, k2 = orc.select_rre(eg, wl.delta)
print("oracle-select on gpu eps == gpu mask:", np.array_equal(m2, mg), k2)
sup = eo > 0
print("eps rel err max", np.max(np.abs(eg[sup]-eo[sup])/eo[sup]), "support equal", np.array_equal(eg > 0, sup))
srt = np.sort(eo)[::-1]; cs = np.cumsum(srt)/srt.sum()
n = mo.sum(); print("oracle prefix at n-1, n:", cs[n-2], cs[n-1], "eps at boundary", srt[n-2:n+1])
d = np.nonzero(mg != mo)[0]
print("eps of diff cells gpu/oracle", eg[d][:6], eo[d][:6])
