"""Full-size, long-run parity where the driver's GPU suite sees it (BASELINE.json north_star: "every
config matches the oracle ... within 1e-10 max relative fp64 state error per conserved variable after
the full run", index lists bit-exact):

* cfg 3: the COMPLETE 500-step run on the full 62,932-cell mesh;
* cfg 5: 20 steps of the full 305,827-cell Navier-Stokes mesh (the complete 200-step run takes
  ~20 min of oracle time on 16 cores: tools/full_run_parity.py 5:200, profiles/);
* cfg 4: 50 steps of the full-size dynamic-AMR run with its 9 device re-meshes.

Each runs tools/full_run_parity.py in a subprocess with the oracle's OpenMP build on every host core
(ORACLE_OMP=1: the parallel loops write disjoint slots, so the oracle's results are bitwise those of
the serial build -- tests/test_oracle_*.py pin the serial one); the GPU side is the C ABI as in every
other GPU test.  The final meshes, faces, per-member lists and stage prefix tables are compared
bitwise, the states per conserved variable."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _full_run(spec):
    env = dict(os.environ, ORACLE_OMP="1", OMP_NUM_THREADS=str(os.cpu_count() or 1))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "full_run_parity.py"), spec],
                         capture_output=True, text=True, env=env, timeout=1500)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout[out.stdout.index("{"):])
    assert res["tolerance"] == 1e-10
    (r,) = res["configs"].values()
    return r


@pytest.mark.parametrize("spec,steps,cells,remeshes", [("3:500", 500, 62932, 0), ("5:20", 20, 305827, 0),
                                                       ("4:50", 50, None, 9)])
def test_full_size_run(spec, steps, cells, remeshes):
    r = _full_run(spec)
    assert r["steps"] == steps and r["re_meshes"] == remeshes
    if cells is not None:
        assert r["cells"] == cells
    assert r["mesh_identical"] and r["lists_identical"], r
    assert max(r["max_rel_err_per_var"]) <= 1e-10, r
    assert r["pass"], r
