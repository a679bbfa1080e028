"""Small runs of every path for compute-sanitizer (memcheck / racecheck / synccheck): the reduced
online step (both PCG kernels), the paper's affine variant, the fine reference scheme and the K6
diagnostics, on C1 and C2 (paper-recipe bases) and a ragged 3D case.  Exits 0 when every run
returns LRBMS_OK."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1405_2810_b200 import inputs  # noqa: E402
from paper_1405_2810_b200.lrbms import LrbmsContext  # noqa: E402

cases = [("C1", lambda: inputs.make_scenario("C1")), ("C2", lambda: inputs.make_scenario("C2")),
         ("ragged3d", lambda: inputs.custom_scenario(9, 6, 4, 3, 3, 2, 11, seed=22, mu_o=10.0,
                                                     bc="corner_columns_3d"))]
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for name, make in cases:
    sc = make()
    for onchip in (1, 0):
        ctx = LrbmsContext(sc, solver={"onchip": onchip})
        ctx.run(steps)
        d = ctx.diagnostics()
        ctx.close()
        print(f"{name} reduced onchip={onchip}: ok, zeta_max {d['zeta_max']:.3e}", flush=True)
    ctx = LrbmsContext(sc)
    ctx.set_profiles(inputs.profile_saturations(sc))
    ctx.set_online(True)
    ctx.run(steps)
    ctx.close()
    print(f"{name} affine: ok", flush=True)
    ctx = LrbmsContext(sc)
    ctx.run_fine(steps, rtol=1e-12)
    ctx.close()
    print(f"{name} fine: ok", flush=True)
torch.cuda.synchronize()
print("all paths ok")
