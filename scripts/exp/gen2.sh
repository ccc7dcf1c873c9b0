# Vessel tree on the GPU vs the host builder: parity tests, time at config 4 and config 5 sizes
timeout 600 python -m pytest tests/test_gpu_tiler.py -q -k "device" 2>&1 | tail -3
python - <<'PY'
import time, sys
sys.path.insert(0, ".")
import torch
from paper_1611_02445_b200 import geometry, tiling
geometry.generate_vessel_tree((64, 64, 64), device=0)   # warm the context
for shape in ((512, 512, 1024), (1024, 1024, 2048)):
    t = time.time(); g = geometry.generate_vessel_tree(shape, device=0); tg = time.time() - t
    t = time.time(); grid = tiling.build_tiling(g); torch.cuda.synchronize(); tt = time.time() - t
    t = time.time(); h = geometry.generate_vessel_tree(shape); th = time.time() - t
    print(shape, "gpu", round(tg, 2), "s cpu", round(th, 2), "s equal", bool((g.types == h.types).all()),
          "tiler", round(tt, 2), "s t_n", grid.t_n, flush=True)
    del g, h, grid
PY
