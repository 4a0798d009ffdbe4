#!/bin/bash
# round 2, call J: the LARGE builder pass (config 1 and dense systems)
cd "$GRAFT_REPO_ROOT"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/j_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cutoff.py tests/test_gpu_md.py -m gpu -q -k "list or drifted or rebuild or half_cells or deferred or overflow or nve or graph or counterexample or ordered" > gpurun_out/j_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/j_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/j_smoke.log
timeout 600 python tools/build_time.py 3,4 > gpurun_out/j_build_time.log 2>&1
python - > gpurun_out/j_c1.log 2>&1 <<'PY'
import json, sys, torch
sys.path.insert(0, ".")
import lj_inputs
from paper_1806_05713_b200 import lj
from tools.build_time import timeit
w = lj_inputs.config(1); g = lj.geom(w.L, w.rc, w.rs)
q = lj.pack_aos4(torch.from_numpy(w.q).cuda())
for half in (False, True):
    b = lj.ListBuilder(w.n, g, half, device="cuda")
    b.build(q)
    print(json.dumps({"cfg": 1, "half": half, "build_ms": round(timeit(lambda: b.build(q)), 4)}))
PY
