"""FFT-size planner over the device transforms (planner.hpp:37-64) and device
postprocessing (pipeline.cpp:60-137), against the compiled reference."""
import numpy as np
import pytest


def _rand_table(rng, lo, hi):
    return {n: float(rng.uniform(1.0, 100.0)) for n in range(lo, hi + 1)}


def test_select_grid_matches_reference(ref):
    import paper_1701_08361_b200 as pb
    rng = np.random.default_rng(5)
    for trial in range(40):
        t = _rand_table(rng, 100, 800)
        if trial % 5 == 0:  # ties resolve toward the smallest G (planner.cpp:122-127)
            for k in t:
                t[k] = 7.0
        N = int(rng.integers(40, 190))
        want = ref.select_grid(N, t)
        got = pb.select_grid(N, pb.FftLookupTable(t))
        assert got[0] == want[0] and got[1] == pytest.approx(want[1], abs=0)
    with pytest.raises(pb.UsageError):
        pb.select_grid(160, pb.FftLookupTable(_rand_table(rng, 100, 400)))  # 640 not covered
    with pytest.raises(pb.UsageError):
        pb.select_grid(160, pb.FftLookupTable(_rand_table(rng, 100, 800)), 1.4, 1.2)


def test_table_files_interchange_with_the_reference(ref, tmp_path):
    import paper_1701_08361_b200 as pb
    t = {n: round(1.0 + 0.37 * n, 3) for n in range(16, 40)}
    pb.save_table(pb.FftLookupTable(t, "b200-sm148", "line-fft"), tmp_path / "ours.tsv")
    back = pb.load_table(tmp_path / "ours.tsv")
    assert back.entries_us == t and back.machine_key == "b200-sm148" and back.library_key == "line-fft"
    assert ref.table_roundtrip(tmp_path / "theirs.tsv", t) == t
    assert pb.load_table(tmp_path / "theirs.tsv").entries_us == t
    (tmp_path / "bad.tsv").write_text("# machine:\tx\n12\tnotanumber\n")
    with pytest.raises(pb.DataError):
        pb.load_table(tmp_path / "bad.tsv")


@pytest.mark.gpu
def test_device_fft_table_drives_the_grid_choice(gpu):
    # every even size of the search window, as select_grid requires (planner.cpp:118-121)
    sizes = list(range(192, 258, 2))
    t = gpu.benchmark_fft(sizes, trials=2, batch=4)
    assert all(v > 0 for v in t.entries_us.values())
    # a size without a fused line engine (200 = 8 x 25) runs the direct DFT and loses
    assert t.entries_us[200] > t.entries_us[256]
    G, gamma = gpu.select_grid(64, t, 1.5, 2.0)
    assert gpu.grid_supported(G) and gamma == G / 128
    p = gpu.plan_from_table(64, 4, t, 1.5, 2.0)
    assert (p.G, p.N, p.Gc) == (G, 64, G // 4)


@pytest.mark.gpu
def test_post_stage_matches_reference(gpu, ref):
    rng = np.random.default_rng(9)
    F, N = 5, 24
    imgs = (rng.standard_normal((F, N, N)) + 1j * rng.standard_normal((F, N, N))).astype(np.complex64)
    mags = np.stack([gpu.magnitude_image(imgs[n]) for n in range(F)])
    want = np.stack([ref.magnitude_image(imgs[n]) for n in range(F)])
    assert np.array_equal(mags, want)
    ph = gpu.phase_difference_image(imgs[0], imgs[1])
    assert np.max(np.abs(ph - ref.phase_difference_image(imgs[0], imgs[1]))) <= 1e-6
    for F_ in (1, 2, 5):
        assert np.array_equal(gpu.median3_sequence(mags[:F_]), ref.median_filter(mags[:F_]))


@pytest.mark.gpu
def test_series_post_on_device_images(gpu, ref):
    plan = gpu.make_plan(16, 2)
    plan.newton_steps, plan.cg_iter_budget = 3, 9
    samples, angles = ref.phantom_series(2, 4, 7, 2, plan.N, 1e-3, 3)
    ctx = gpu.Context(plan)
    s = gpu.Series(ctx, 4, 2)
    out = s.run(gpu.SeriesOptions(plain=True), raw=dict(samples=samples, angles=angles))
    mags = np.stack([ref.magnitude_image(out["images"][n]) for n in range(4)])
    assert np.array_equal(s.post(mode="magnitude"), mags)
    assert np.array_equal(s.post(mode="median3"), ref.median_filter(mags))
    pd = s.post(mode="phase_difference")
    assert pd.shape == (2, plan.N, plan.N)
    assert np.max(np.abs(pd[1] - ref.phase_difference_image(out["images"][2], out["images"][3]))) <= 1e-6
