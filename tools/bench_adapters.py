"""Per-call cost of the drop-in adapters against the reference functions they replace (tetris_sched from
baseline/_ref), on the same inputs, with the reference's results compared for equality.  Prints one JSON line.
usage: python tools/bench_adapters.py"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))


def timed(fn, reps):
    fn()  # warm (first call: CUDA context, workspaces)
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    return (time.perf_counter() - t0) / reps * 1e3, out


def main():
    import tetris_sched.accept_model as RA
    import tetris_sched.selector as RS
    import tetris_sched.sim_engine as RE

    from paper_2502_15197_b200 import accept_model as GA
    from paper_2502_15197_b200 import dropin
    from paper_2502_15197_b200 import selector as GS
    from paper_2502_15197_b200 import sim_engine as GE

    rng = np.random.default_rng(0)
    res = {}
    ref = {n: getattr(m, n) for m, names in ((RS, ("cumulative_products", "select_tetris")),
                                              (RA, ("verify_token", "residual_distribution"))) for n in names}
    inst = dropin.install(RS, RA, RE)  # the adapters build the reference's own classes
    try:
        for B, k, C in ((16, 5, 48), (1024, 16, 8192)):
            rows = [tuple(float(x) for x in rng.random(k) ** 0.25) for _ in range(B)]
            mat = RA.AcceptanceMatrix(tuple(rows))
            t_ref_c, cand_ref = timed(lambda: ref["cumulative_products"](mat), 3)
            t_gpu_c, cand = timed(lambda: GS.cumulative_products(mat), 3)
            t_ref_s, (sel_ref, st_ref) = timed(lambda: ref["select_tetris"](cand_ref, C), 3)
            t_gpu_s, (sel, st) = timed(lambda: GS.select_tetris(cand, C), 3)
            t_gpu_sf, (sel_f, _) = timed(lambda: GS.select_tetris(cand, C, exact_stats=False), 3)
            res[f"B={B} k={k} C={C}"] = {
                "cumulative_products_ms": {"reference": t_ref_c, "adapter": t_gpu_c},
                "select_tetris_ms": {"reference": t_ref_s, "adapter": t_gpu_s, "adapter_closed_form_stats": t_gpu_sf},
                "equal": bool(sel == sel_ref and st == st_ref and sel_f == sel_ref)}
        V = 128256
        pd = rng.random(V)
        pt = rng.random(V)
        dd = RA.TokenDistribution(pd / pd.sum())
        dt = RA.TokenDistribution(pt / pt.sum())
        t_ref_v, a_ref = timed(lambda: ref["verify_token"](dd, dt, 17, 0.3), 20)
        t_gpu_v, a = timed(lambda: GA.verify_token(dd, dt, 17, 0.3), 20)
        t_ref_r, r_ref = timed(lambda: ref["residual_distribution"](dd, dt), 5)
        t_gpu_r, r = timed(lambda: GA.residual_distribution(dd, dt), 5)
        res["V=128256"] = {"verify_token_ms": {"reference": t_ref_v, "adapter": t_gpu_v},
                           "residual_distribution_ms": {"reference": t_ref_r, "adapter": t_gpu_r},
                           "equal_verify": bool(a == a_ref),
                           "residual_max_abs_diff": float(np.max(np.abs(np.asarray(r.probs) - np.asarray(r_ref.probs))))}
    finally:
        inst.uninstall()
    print(json.dumps({"what": "drop-in adapters vs the reference functions, per call (ms)", "results": res}))


if __name__ == "__main__":
    main()
