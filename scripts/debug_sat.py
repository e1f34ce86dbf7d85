import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, "."); sys.path.insert(0, "oracle")
from conftest import load_case, scene_from
from paper_2602_22625_b200 import raster, grad
import cpu_oracle as orc
d = load_case("saturated"); sc = scene_from(d)
np.set_printoptions(precision=6, linewidth=200)
for eps, key_dI, key_g in ((1/1024, "dI", "grads"), (0.0, "dI_eps0", "grads_eps0")):
    out, saved = raster.render_forward(sc, save=True, eps_skip=eps)
    g = grad.backward(sc, saved, d[key_dI])
    print("eps", eps, "n_entries", saved.n_entries)
    print("gpu ", g.data)
    print("ref ", d[key_g])
    pk = orc.Packed(sc); off, idx = orc.bin_tiles(pk, 16, 2.0)
    img, a, sv = orc.render_forward(pk, off, idx, 16, orc.background(sc), True, eps)
    print("orc ", orc.backward(pk, sv, d[key_dI], None))
    print("ent_n gpu", saved.compositor.ent_n.view(24,24).cpu().numpy().sum(), "orc", sv["n_entries"])
