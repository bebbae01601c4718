cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do for k in tc cuda; do echo -n "ks=$k "; GATEWAVE_KS_KERNEL=$k timeout 300 python tools/c2_time.py 2>/dev/null | tail -1; done; done
GATEWAVE_BR_PROFILE=0 timeout 300 python - <<'PY'
import sys, numpy as np, time
sys.path.insert(0, '.')
from paper_2306_11006_b200.cggi import PARAM_128, keygen
from paper_2306_11006_b200 import engine as E
import os
ks = keygen(PARAM_128, seed=7)
for kern in ("tc", "cuda"):
    os.environ["GATEWAVE_KS_KERNEL"] = kern
    eng = E.Engine(*E.params_tuple(PARAM_128)); eng.upload_keys(ks.bootstrapping_key.data, ks.keyswitch_key.data)
    for U in (1, 2, 4, 8, 16, 32, 64, 128, 256):
        ext = np.random.default_rng(U).integers(0, 2**32, (U, PARAM_128.N + 1), dtype=np.uint32)
        eng.set_profiling(True); eng.stage_times(reset=True)
        for _ in range(20): eng.keyswitch(ext)
        st = eng.stage_times(reset=True); eng.set_profiling(False)
        print(kern, U, {k: round(v[0] / 20 * 1e6, 1) for k, v in st.items()})
PY
