"""Evaluation-path cases (metrics.py) shared by make_golden_metrics.py and the tests.

``build(case, O, ref=None)`` returns (original axes, reconstructed axes,
CompressConfig kwargs).  The reconstruction is compress -> decompress of
the original (the reference when ``ref`` is given, else the oracle, which is
pinned byte-for-byte to it) followed by the case's deterministic edit.
"""

import numpy as np

METRIC_CASES = [
    dict(name="clusters3_f32_rel", gen="clusters", count=5000, dims=3, dt="f32", seed=11, eb=1e-3, mode=1),
    dict(name="uniform2_f64_abs", gen="uniform", count=3000, dims=2, dt="f64", seed=12, eb=1e-4, mode=0),
    dict(name="lattice1_f32_bs256", gen="lattice", count=2500, dims=1, dt="f32", seed=13, eb=1e-2, mode=1,
         bs=256, t=8),
    dict(name="clusters3_perturbed", gen="clusters", count=4096, dims=3, dt="f32", seed=14, eb=1e-3, mode=1,
         edit="perturb"),
    dict(name="clusters3_rec_f64", gen="clusters", count=3000, dims=3, dt="f32", seed=15, eb=1e-3, mode=1,
         edit="as_f64"),
    dict(name="uniform3_reversed", gen="uniform", count=2048, dims=3, dt="f32", seed=16, eb=1e-2, mode=1,
         edit="reverse_blocks"),
    dict(name="constant3", gen="constant", count=1500, dims=3, dt="f32", seed=17, eb=1e-3, mode=1),
    dict(name="partial_tail_f64", gen="clusters", count=2100, dims=2, dt="f64", seed=18, eb=1e-5, mode=1,
         bs=512, t=16, edit="perturb"),
    dict(name="err_shape", gen="clusters", count=1000, dims=3, dt="f32", seed=19, eb=1e-3, mode=1,
         edit="truncate"),
    dict(name="err_nonfinite_rec", gen="clusters", count=1000, dims=3, dt="f32", seed=20, eb=1e-3, mode=1,
         edit="nan"),
    dict(name="err_width", gen="huge", count=64, dims=1, dt="f64", seed=21, eb=1e-300, mode=0),
]


def _orig(case, O):
    dt = O.F32 if case["dt"] == "f32" else O.F64
    npdt = np.float32 if case["dt"] == "f32" else np.float64
    g, n, d, seed = case["gen"], case["count"], case["dims"], case["seed"]
    if g == "clusters":
        return O.gen_clusters(n, d, seed=seed, prec=dt)
    if g == "uniform":
        return O.gen_uniform(n, d, seed=seed, prec=dt)
    if g == "lattice":
        return O.gen_lattice(n, d, seed=seed, prec=dt)
    if g == "constant":
        return [np.full(n, 0.25 * (a + 1), npdt) for a in range(d)]
    if g == "huge":
        return [np.linspace(0.0, 1e300, n).astype(npdt) for _ in range(d)]
    raise ValueError(g)


def cfg_kwargs(case):
    return dict(error_bound=case["eb"], eb_mode=case["mode"], block_size=case.get("bs", 1024),
                target_segs_per_axis=case.get("t", 32))


def build(case, O, ref=None):
    orig = _orig(case, O)
    kw = cfg_kwargs(case)
    if case["name"] == "err_width":
        rec = [a.copy() for a in orig]
    elif ref is not None:
        cfg = ref.CompressConfig(error_bound=kw["error_bound"], eb_mode=ref.EbMode(kw["eb_mode"]),
                                 block_size=kw["block_size"], target_segs_per_axis=kw["target_segs_per_axis"])
        rec = [np.array(a) for a in ref.decompress(ref.compress(ref.Dataset.from_axes(orig), cfg)).axes]
    else:
        cfg = O.Config(kw["error_bound"], eb_mode=kw["eb_mode"], block_size=kw["block_size"],
                       target_segs_per_axis=kw["target_segs_per_axis"])
        rec = [np.array(a) for a in O.decompress(O.compress(orig, cfg))]
    edit = case.get("edit")
    if edit == "perturb":
        eb_abs = O.absolute_bound(orig, O.Config(kw["error_bound"], eb_mode=kw["eb_mode"]))
        n = orig[0].size
        for j, (i, a) in enumerate([(5, 0), (n // 3, 1 % case["dims"]), (n // 2, 0), (n - 1, case["dims"] - 1)]):
            rec[a][i] = rec[a][i] + (3.0 + j) * eb_abs
    elif edit == "as_f64":
        rec = [a.astype(np.float64) + 1e-7 for a in rec]
    elif edit == "reverse_blocks":
        bs = kw["block_size"]
        rec = [np.concatenate([a[s:s + bs][::-1] for s in range(0, a.size, bs)]) for a in rec]
    elif edit == "truncate":
        rec = [a[:-1].copy() for a in rec]
    elif edit == "nan":
        rec[1][17] = np.nan
    return orig, rec, kw
