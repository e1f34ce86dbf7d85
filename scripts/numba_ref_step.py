"""Time the UNMODIFIED reference (numba primfit from baseline/_ref) on its own
run_loop body, SURVEY.md §8(d) CPU protocol: NUMBA_NUM_THREADS = all host cores,
warmup_kernels() + one untimed step, then the median of the timed steps of
unpack_params -> bin_tiles(tile 32) -> render_forward(save) -> evaluate_loss ->
backward -> adam_step -> psnr (fit.py:479-505).

    python scripts/numba_ref_step.py c3 [max_steps] [max_seconds]

Prints one JSON object.  Used by bench.py as a second CPU reading next to the
C/OpenMP port (run in a subprocess so the numba thread pool owns the cores).
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
os.environ.setdefault("NUMBA_NUM_THREADS", str(os.cpu_count() or 1))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
sys.path.insert(0, str(ROOT))


def main() -> None:
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    max_steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    max_seconds = float(sys.argv[3]) if len(sys.argv) > 3 else 15.0
    import numba
    import numpy as np
    from primfit import fit as rfit
    from primfit import raster as rr
    from primfit import grad as rgrad
    from primfit.scene import PrimitiveParams, PrimitiveTemplate, Scene, pack_params, unpack_params

    from paper_2602_22625_b200 import synth

    w = synth.make_workload(name)
    sc = Scene([PrimitiveParams(x=p.x, y=p.y, scale=p.scale, rotation=p.rotation,
                                opacity_logit=p.opacity_logit, color_logits=tuple(p.color_logits),
                                template_id=p.template_id, z=p.z) for p in w.scene.primitives],
               [PrimitiveTemplate(np.asarray(t.rgba)) for t in w.scene.templates],
               canvas_w=w.scene.canvas_w, canvas_h=w.scene.canvas_h,
               background=tuple(w.scene.background))
    cfg = w.cfg
    spec = rfit.LossSpec(kind="mse", target=w.target)
    t_jit = time.perf_counter()
    rr.warmup_kernels()
    jit_s = time.perf_counter() - t_jit
    vec, layout = pack_params(sc)
    state = rfit.OptimState.fresh(layout)
    gains = rfit.gains_vector(layout, {"x": cfg.lr_gain_x, "y": cfg.lr_gain_y,
                                       "scale": cfg.lr_gain_scale,
                                       "rotation": cfg.lr_gain_rotation,
                                       "opacity": cfg.lr_gain_opacity,
                                       "color": cfg.lr_gain_color})
    padding = rfit.effective_padding(cfg)
    total = w.steps

    def body(it, vec, scene):
        lr = rfit.lr_schedule(it, total, cfg.learning_rate, cfg.do_decay,
                              cfg.decay_final_fraction)
        scene = unpack_params(vec, layout, scene)
        bins = rr.bin_tiles(scene, 32, padding)
        out, saved = rr.render_forward(scene, bins, None, save=True, eps_skip=cfg.eps_skip)
        value, dI, dA = rfit.evaluate_loss(spec, out.color, out.alpha)
        grads = rgrad.backward(scene, saved, dI, dA)
        vec = rfit.adam_step(vec, grads.to_vector(), state, lr, gains, s_min=cfg.scale_min,
                             s_max=cfg.scale_max, layout=layout)
        rfit.psnr(out.color, spec.target)
        return vec, scene

    vec, sc = body(0, vec, sc)  # untimed
    times = []
    t_all = time.perf_counter()
    it = 1
    while it < total and len(times) < max_steps and time.perf_counter() - t_all < max_seconds:
        t0 = time.perf_counter()
        vec, sc = body(it, vec, sc)
        times.append(time.perf_counter() - t0)
        it += 1
    med = float(np.median(times))
    print(json.dumps({
        "value": 1.0 / med, "unit": "steps/s", "cores": numba.get_num_threads(),
        "kind": "reference",
        "sample": f"{name}: median of {len(times)} run_loop-body steps of the unmodified numba "
                  f"reference (baseline/_ref) after warmup_kernels + 1 untimed step",
        "ms_per_step": med * 1e3, "threading_layer": numba.threading_layer(),
        "jit_s": jit_s}))


if __name__ == "__main__":
    main()
