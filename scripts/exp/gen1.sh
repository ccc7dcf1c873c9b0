timeout 600 python -m pytest tests/test_gpu_tiler.py -q -k device 2>&1 | tail -3
python - <<'PY'
import time, sys
sys.path.insert(0, ".")
from paper_1611_02445_b200 import geometry
for n, p in ((256, 0.2), (512, 0.5), (1024, 0.5)):
    t = time.time(); g = geometry.generate_sphere_pack(n, 40, p, 1234, device=0); tg = time.time() - t
    if n <= 512:
        t = time.time(); h = geometry.generate_sphere_pack(n, 40, p, 1234); th = time.time() - t
        print(n, p, "gpu", round(tg, 2), "s cpu", round(th, 2), "s equal", (g.types == h.types).all())
    else:
        print(n, p, "gpu", round(tg, 2), "s porosity", g.porosity())
PY
