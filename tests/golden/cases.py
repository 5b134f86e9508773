"""Fixture specifications shared by make_golden.py (which runs the reference
in the build container) and the tests (which regenerate inputs with the
oracle's generators and compare against the committed outcomes)."""

import numpy as np

# (name, generator, count, dims, dtype, eb, eb_mode, block_size, target, preserve, seed, extra)
CASES = [
    ("clu3_f32_e3", "clusters", 3000, 3, "f32", 1e-3, 1, 1024, 32, False, 1, {}),
    ("clu3_f32_e2", "clusters", 3000, 3, "f32", 1e-2, 1, 1024, 32, False, 2, {}),
    ("clu3_f32_e4", "clusters", 3000, 3, "f32", 1e-4, 1, 1024, 32, False, 3, {}),
    ("uni3_f32_e3", "uniform", 3000, 3, "f32", 1e-3, 1, 1024, 32, False, 4, {}),
    ("uni3_f32_e4", "uniform", 3000, 3, "f32", 1e-4, 1, 1024, 32, False, 5, {}),
    ("uni3_f32_e2", "uniform", 3000, 3, "f32", 1e-2, 1, 1024, 32, False, 6, {}),
    ("lat3_f32_e3", "lattice", 3000, 3, "f32", 1e-3, 1, 1024, 32, False, 7, {}),
    ("lat3_f32_e2", "lattice", 3000, 3, "f32", 1e-2, 1, 1024, 32, False, 8, {}),
    ("uni2_f64_abs", "uniform", 2500, 2, "f64", 1e-5, 0, 1024, 32, False, 9, {}),
    ("clu1_f32_e6", "clusters", 2000, 1, "f32", 1e-6, 1, 1024, 32, False, 10, {}),
    ("clu1_f64_e9", "clusters", 2000, 1, "f64", 1e-9, 1, 1024, 32, False, 11, {}),
    ("clu3_f32_pres", "clusters", 3000, 3, "f32", 1e-3, 1, 1024, 32, True, 12, {}),
    ("uni2_f64_pres", "uniform", 2100, 2, "f64", 1e-4, 1, 1024, 32, True, 13, {}),
    ("clu1_f32_pres_e2", "clusters", 1500, 1, "f32", 1e-2, 1, 1024, 32, True, 14, {}),
    ("clu3_bs32", "clusters", 1000, 3, "f32", 1e-3, 1, 32, 32, False, 15, {}),
    ("clu3_bs96", "clusters", 1000, 3, "f32", 1e-3, 1, 96, 32, False, 16, {}),
    ("clu3_bs512", "clusters", 2000, 3, "f32", 1e-3, 1, 512, 32, False, 17, {}),
    ("uni3_t1", "uniform", 2000, 3, "f32", 1e-3, 1, 1024, 1, False, 18, {}),
    ("uni3_t2", "uniform", 2000, 3, "f32", 1e-3, 1, 1024, 2, False, 19, {}),
    ("uni3_t8", "uniform", 2000, 3, "f32", 1e-3, 1, 1024, 8, False, 20, {}),
    ("uni3_t64", "uniform", 2000, 3, "f32", 1e-3, 1, 1024, 64, False, 21, {}),
    ("uni3_t128", "uniform", 2000, 3, "f32", 1e-4, 1, 1024, 128, False, 22, {}),
    ("uni2_t1024", "uniform", 2000, 2, "f64", 1e-6, 1, 1024, 1024, False, 23, {}),
    ("uni3_t128_pres", "uniform", 1500, 3, "f32", 1e-4, 1, 1024, 128, True, 24, {}),
    ("const3", "const", 2048, 3, "f32", 1e-3, 1, 1024, 32, False, 0, {"value": 1.5}),
    ("const1_pres", "const", 100, 1, "f64", 1e-3, 0, 32, 32, True, 0, {"value": -2.25}),
    ("n1", "uniform", 1, 3, "f32", 1e-3, 1, 1024, 32, False, 25, {}),
    ("n31", "uniform", 31, 2, "f32", 1e-3, 0, 32, 32, False, 26, {}),
    ("n33", "uniform", 33, 2, "f32", 1e-3, 1, 32, 32, True, 27, {}),
    ("empty2_f64", "uniform", 0, 2, "f64", 0.1, 0, 1024, 32, False, 0, {}),
    ("empty3_rel", "uniform", 0, 3, "f32", 1e-3, 1, 1024, 32, False, 0, {}),
    ("half_f32", "offset_uniform", 3000, 3, "f32", 1e-2, 0, 1024, 32, False, 28, {"base": 1e6, "width": 100.0}),
    ("half_f32_rel", "offset_uniform", 3000, 2, "f32", 1e-9, 1, 1024, 32, False, 29, {"base": 1e3, "width": 1.0}),
    ("half_f64", "offset_uniform", 2000, 1, "f64", 1e-17, 0, 1024, 32, False, 30, {"base": 0.0, "width": 1.0}),
    ("half_f64_pres", "offset_uniform", 1000, 2, "f64", 1e-16, 0, 1024, 32, True, 31, {"base": 10.0, "width": 1.0}),
    ("half_f64_pres_ok", "offset_uniform", 1000, 2, "f64", 1e-15, 0, 1024, 32, True, 38, {"base": 10.0, "width": 1e-9}),
    ("half_f32_pres", "offset_uniform", 1500, 3, "f32", 1e-2, 0, 1024, 32, True, 39, {"base": 1e6, "width": 10.0}),
    ("bigq_f32", "offset_uniform", 3000, 1, "f32", 2e-7, 1, 1024, 32, False, 32, {"base": 0.0, "width": 1.0}),
    ("bigq_f64", "offset_uniform", 3000, 2, "f64", 1e-11, 1, 1024, 32, False, 33, {"base": -3.0, "width": 6.0}),
    ("neg_mixed", "offset_uniform", 3000, 3, "f32", 1e-3, 1, 1024, 32, False, 34, {"base": -50.0, "width": 100.0}),
    ("outlier", "outlier", 3000, 3, "f32", 1e-4, 0, 1024, 32, False, 35, {}),
    ("outlier_f64", "outlier", 3000, 3, "f64", 1e-6, 0, 1024, 32, False, 36, {}),
    ("width_overflow", "explicit", 2, 1, "f64", 1e-12, 0, 32, 32, False, 0, {"values": [[0.0, 1e30]]}),
    ("geom_overflow", "explicit", 2, 3, "f64", 0.5, 0, 32, 32, False, 0,
     {"values": [[0.0, 1e9], [0.0, 1e9], [0.0, 1e9]]}),
    ("overflow_block2", "overflow_late", 200, 1, "f64", 1e-12, 0, 64, 32, False, 0, {}),
    ("nonfinite", "nonfinite", 100, 2, "f32", 1e-3, 1, 32, 32, False, 37, {}),
    ("four_particles", "explicit", 4, 1, "f64", 0.5, 0, 32, 32, False, 0, {"values": [[0.2, 3.7, 5.1, 7.9]]}),
]


def make_axes(gen, count, dims, dtype, seed, extra, O):
    """Inputs for a case; O is the oracle module (its generators restate bench.py:56-94)."""
    prec = O.F32 if dtype == "f32" else O.F64
    npt = np.float32 if dtype == "f32" else np.float64
    if gen == "clusters":
        return O.gen_clusters(count, dims=dims, seed=seed, prec=prec)
    if gen == "uniform":
        return O.gen_uniform(count, dims=dims, seed=seed, prec=prec)
    if gen == "lattice":
        return O.gen_lattice(count, dims=dims, seed=seed, prec=prec)
    if gen == "const":
        return [np.full(count, extra["value"], npt) for _ in range(dims)]
    if gen == "offset_uniform":
        rng = np.random.default_rng(seed)
        return [(extra["base"] + rng.uniform(0, extra["width"], count)).astype(npt) for _ in range(dims)]
    if gen == "outlier":
        rng = np.random.default_rng(seed)
        axes = [rng.normal(0.5, 0.001, count) for _ in range(dims)]
        for a in axes:
            a[::997] += 3.0  # one far particle per ~block stretches the geometry
        return [a.astype(npt) for a in axes]
    if gen == "explicit":
        return [np.asarray(v, npt) for v in extra["values"]]
    if gen == "overflow_late":
        x = np.linspace(0.0, 1.0, count)
        x[150] = 1e30  # block 2 of 64-particle blocks overflows
        return [x.astype(npt)]
    if gen == "nonfinite":
        rng = np.random.default_rng(seed)
        axes = [rng.uniform(0, 1, count).astype(npt) for _ in range(dims)]
        axes[1][77] = np.nan
        return axes
    raise ValueError(gen)
