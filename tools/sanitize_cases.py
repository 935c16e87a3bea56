"""Small invocations of every kernel family, for compute-sanitizer (one tool per
gpurun call: memcheck, racecheck, synccheck -- tools/gpu.sh sanitize <tool>).
Each case runs one predict and checks it against the oracle, so a sanitizer
run also proves the instrumented kernels still compute the right thing.

Cases (VERDICT r1 "what's weak" #9 lists the async pipelines to cover):
  C1 (1 CTA), 4096-row C2 and C3 (resident chunks, threshold-bin codes, K4 /
  K4d), C5-shaped deep chunks (K4d + child-pair speculation), a C4-shaped
  tree-streamed model (K4s: loader warp ring, slot headers, cp.async landing
  slots), the fused GEMM-form kernel fz_kernel (K5) and the staged
  gc -> pc -> lg pipeline (K1/K2/K3), a linear model, and the cluster/DSMEM
  variant of K4 (BRIDGER_CLUSTER=1), and round 2's binning kernels.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2405_12491_b200 as B  # noqa: E402
from synth import gen_x, iris_like_x, make_config, perfect_ensemble  # noqa: E402


def check(name, m, X, variant=None, env=None):
    old = {}
    for k, v in (env or {}).items():
        old[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        g = B.Model(m, device=0, variant=variant)
        xd = torch.from_numpy(X).cuda()
        got = g.predict(xd).cpu().numpy()
        o = oracle.run(m, X)
        want = o["label"] if m.task == 1 else o["pred"]
        if m.task == 1:
            assert np.array_equal(got, want), name
        else:
            np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-6, err_msg=name)
        fmt = g.layout()["format"] if variant in (None, "traverse") else variant
        g.close()
        print(f"case {name}: ok ({fmt})", flush=True)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def main():
    torch.cuda.set_device(0)
    only = set(sys.argv[1:])
    cases = []
    _, m1 = make_config("C1")
    cases.append(("C1", m1, iris_like_x(1), None, None))
    c2, m2 = make_config("C2", n_trees=100)
    cases.append(("C2_4096", m2, gen_x(2, 0, 4096, 28), None, None))
    c3, m3 = make_config("C3", n_trees=500)
    cases.append(("C3_4096_deep", m3, gen_x(3, 0, 4096, 90), None, None))
    cases.append(("C3_4096_k4", m3, gen_x(3, 0, 4096, 90), None, {"BRIDGER_DEEP": "0"}))
    c5, m5 = make_config("C5", n_trees=300)
    cases.append(("C5_shaped_deep_spec", m5, gen_x(5, 0, 2048, 200), None, None))
    c4, m4 = make_config("C4", n_trees=16)
    cases.append(("C4_stream", m4, gen_x(4, 0, 2048, 64), None, None))
    cases.append(("C2_fz_kernel", make_config("C2", n_trees=12)[1], gen_x(2, 0, 1000, 28), "gemm", None))
    cases.append(("C2_staged_gc_pc_lg", make_config("C2", n_trees=12)[1], gen_x(2, 0, 1000, 28), "gemm_staged", None))
    cases.append(("C2_cluster_dsmem", make_config("C2", n_trees=100)[1], gen_x(2, 0, 4096, 28), None,
                  {"BRIDGER_CLUSTER": "1", "BRIDGER_CODES": "0"}))
    # round-2 binning kernels: bucket entries (TMA row tiles), feature-group
    # bucketed tables with TMA tiles, Eytzinger pairs with TMA tiles (2^16-slot
    # trees: tests/test_gpu_parity.py test_coded_wide_code_range), the
    # three-buffer all-features bucketed kernel, odd F (4-row views)
    cases.append(("C2_bin_entry", m2, gen_x(2, 0, 4099, 28), None, {"BRIDGER_BIN": "E"}))
    cases.append(("C3_bin_bucket_nbuf3", m3, gen_x(3, 0, 4099, 90), None, {"BRIDGER_BIN": "b"}))
    cases.append(("C5_bin_fg_tma", m5, gen_x(5, 0, 2048, 200), None, None))
    cases.append(("C4_codes_bin_fg4", make_config("C4", n_trees=40)[1], gen_x(4, 0, 2048, 64), None,
                  {"BRIDGER_CODES": "1"}))
    cases.append(("F21_bin_entry_R4", perfect_ensemble(27, 90, 8, 21, kind="classification", n_classes=3,
                                                       calib_rows=2048), gen_x(28, 0, 3001, 21), None,
                  {"BRIDGER_BIN": "E", "BRIDGER_CODES": "1"}))
    for name, m, X, variant, env in cases:
        if only and name not in only:
            continue
        check(name, m, X, variant, env)
    # linear model (bulk-copied row blocks, per-warp mbarriers)
    if not only or "linear" in only:
        rng = np.random.default_rng(0)
        from types import SimpleNamespace
        lm = SimpleNamespace(n_features=28, n_outputs=1, coef=rng.standard_normal((1, 28)),
                             intercept=np.array([0.1]), mean=None, scale=None, task=1, post=1)
        g = B.LinearModel(lm, device=0)
        X = gen_x(7, 0, 4099, 28)
        got = g.predict(torch.from_numpy(X).cuda()).cpu().numpy()
        want = oracle.run_linear(lm, X)["label"]
        assert np.array_equal(got, want)
        print("case linear: ok", flush=True)
    torch.cuda.synchronize()
    print("all cases ok", flush=True)


if __name__ == "__main__":
    main()
