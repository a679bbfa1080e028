"""A/B of library variants on one scenario: builds the scenario once (pickled), then times the step and
its stages with every library given (subprocesses, LRBMS_LIB).
usage: python tools/exp_ab.py C5 poly 50 paper_1405_2810_b200/liblrbms.so variants/x.so ..."""
import json
import os
import pickle
import subprocess
import sys

sys.path.insert(0, ".")

if sys.argv[1] == "--child":
    import torch
    from paper_1405_2810_b200.lrbms import LrbmsContext
    sc = pickle.load(open(sys.argv[2], "rb"))
    n = int(sys.argv[3])
    ctx = LrbmsContext(sc)
    if os.environ.get("EXP_AFFINE"):   # the paper's affine online variant (NEXT-1)
        from paper_1405_2810_b200 import inputs
        ctx.set_profiles(inputs.profile_saturations(sc))
        ctx.set_online(True)
    if os.environ.get("EXP_FINE"):   # the fine reference scheme (NEXT-2): ms per step, CG iterations
        ctx.run_fine(1, rtol=1e-12)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(ctx.stream)
        _, its = ctx.run_fine(n, rtol=1e-12)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        print(json.dumps({"lib": os.environ.get("LRBMS_LIB", "default"), "fine_ms_per_step": round(ms, 3),
                          "cg_iters_per_step": its / n, "us_per_iter": round(1e3 * ms / (its / n), 2)}), flush=True)
        sys.exit(0)
    ctx.run(5)
    s0 = ctx.stats()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(ctx.stream)
    ctx.run(n)
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    wall = e0.elapsed_time(e1) / n
    s1 = ctx.stats()
    ctx.set_saturation(sc.s0)
    ctx.run(5)
    ctx.set_profiling(True)
    ctx.run(n)
    st = ctx.stage_times()
    print(json.dumps({"lib": os.environ.get("LRBMS_LIB", "default"), "ms_per_step": round(wall, 4),
                      "iters": (s1["total_iters"] - s0["total_iters"]) / n,
                      **{k: round(1e3 * v[0] / n, 1) for k, v in st.items()}}), flush=True)
    sys.exit(0)

from paper_1405_2810_b200 import inputs  # noqa: E402
cfg, basis, n = sys.argv[1], sys.argv[2], sys.argv[3]
sc = inputs.make_scenario(cfg, basis=basis)
path = f"/tmp/sc_{cfg}_{basis}.pkl"
pickle.dump(sc, open(path, "wb"))
for rep in range(2):
    for lib in sys.argv[4:]:
        env = dict(os.environ, LRBMS_LIB=os.path.abspath(lib))
        subprocess.run([sys.executable, __file__, "--child", path, n], env=env)
