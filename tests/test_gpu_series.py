"""Series drivers on the device: plain chaining, temporal decomposition (T frames in
flight on one B200), the end-to-end host-streaming path, and audit-replay parity
against the compiled reference (SURVEY.md §7 "audit replay")."""
import numpy as np
import pytest

from helpers import rel_err

pytestmark = pytest.mark.gpu

FRAME_TOL = 1e-3


def _series_inputs(ref, plan, F, K, U, noise=1e-4, seed=11):
    samples, angles = ref.phantom_series(plan.J, F, K, U, plan.N, noise, seed)
    z = np.stack([ref.grid_adjoint(plan, samples[n], angles[n]) for n in range(F)])
    # a K-spoke U-turn trajectory revisits its angle set every U frames
    P = np.stack([ref.build_psf(plan, angles[n], 2 * plan.N) for n in range(min(U, F))])
    idx = [n % U for n in range(F)]
    return samples, angles, z, P, idx


def _small_plan(gpu, N, J, M, budget):
    plan = gpu.make_plan(N, J)
    plan.newton_steps, plan.cg_iter_budget = M, budget
    return plan


def _run(gpu, plan, z, P, idx, opts, **kw):
    ctx = gpu.Context(plan)
    s = gpu.Series(ctx, z.shape[0], P.shape[0])
    s.upload_frames(z)
    for k in range(P.shape[0]):
        s.upload_psf(k, P[k])
    s.set_psf_index(idx)
    out = s.run(opts, **kw)
    out["series"], out["ctx"] = s, ctx
    return out


def test_plain_series_matches_reference(gpu, ref):
    plan = _small_plan(gpu, 24, 3, 7, 30)
    samples, angles, z, P, idx = _series_inputs(ref, plan, F=6, K=11, U=5)
    want = ref.reconstruct_series(plan, samples, angles, plain=True)
    got = _run(gpu, plan, z, P, idx, gpu.SeriesOptions(plain=True))
    for n in range(6):
        assert rel_err(got["images"][n], want["images"][n]) < FRAME_TOL, n
        a = got["audit"][n]
        assert a.init_src == want["audit"][n][3] and a.reg_final_src == want["audit"][n][4]
    assert list(got["cg_iters"]) == list(want["cg_iters"])


def test_one_scheduled_thread_reproduces_plain_bit_for_bit(gpu, ref):
    # test_decomp.cpp:328-343
    plan = _small_plan(gpu, 16, 3, 3, 6)
    _, _, z, P, idx = _series_inputs(ref, plan, F=6, K=5, U=3)
    plain = _run(gpu, plan, z, P, idx, gpu.SeriesOptions(plain=True, sched=gpu.TemporalSchedule.for_turns(3)))
    sched = _run(gpu, plan, z, P, idx, gpu.SeriesOptions(T=1, sched=gpu.TemporalSchedule.for_turns(3)))
    assert np.array_equal(plain["images"], sched["images"])
    for a, b in zip(plain["audit"], sched["audit"]):
        assert (a.init_src, a.reg_final_src) == (b.init_src, b.reg_final_src)


@pytest.mark.parametrize("T", [2, 4])
def test_scheduled_threads_keep_the_ordering_contract_and_replay_exactly(gpu, ref, T):
    # test_decomp.cpp:345-387, then every frame replayed through the reference with
    # the sources its audit recorded
    plan = _small_plan(gpu, 16, 3, 3, 6)
    F = 8
    _, _, z, P, idx = _series_inputs(ref, plan, F=F, K=5, U=3)
    sched = gpu.TemporalSchedule(2, 2)
    out = _run(gpu, plan, z, P, idx, gpu.SeriesOptions(T=T, sched=sched))
    M = plan.newton_steps
    audit = out["audit"]
    for n in range(F):
        a = audit[n]
        assert a.frame == n
        assert np.sum(np.abs(out["images"][n]) ** 2) > 0
        if n == 0:
            assert a.init_src == -1
            continue
        assert 0 <= a.init_src < n
        for m in range(M):
            assert 0 <= a.reg_src[m] < n
            if n > sched.l and m < M - 1:
                assert a.reg_src[m] >= n - sched.o
        assert a.reg_final_src == n - 1
        assert a.reg_final_seq > audit[n - 1].finish_seq
        if n <= sched.l:
            assert a.start_seq > audit[n - 1].finish_seq
    # replay: the data were normalised on the device with the series scale
    scale = out["series"].normalize()
    zs = (z * np.float32(scale)).astype(np.complex64)
    unity = gpu.initial_estimate(plan)
    ests = {}
    for n in range(F):
        a = audit[n]
        init = unity if a.init_src < 0 else ests[a.init_src]
        regs = [unity if a.init_src < 0 else ests[a.reg_src[m]] for m in range(M)]
        img, est, _ = ref.reconstruct_frame_regs(plan, zs[n], P[idx[n]], init, regs)
        ests[n] = est
        img = img * np.float32(1.0 / scale)
        assert rel_err(out["images"][n], img) < FRAME_TOL, n
        assert rel_err(out["series"].estimate(n), est) < FRAME_TOL, n


def test_host_streaming_path_equals_resident_path(gpu, ref):
    plan = _small_plan(gpu, 24, 3, 7, 30)
    _, _, z, P, idx = _series_inputs(ref, plan, F=5, K=11, U=5)
    resident = _run(gpu, plan, z, P, idx, gpu.SeriesOptions(plain=True))
    ctx = gpu.Context(plan)
    s = gpu.Series(ctx, 5, P.shape[0])
    for k in range(P.shape[0]):
        s.upload_psf(k, P[k])
    s.set_psf_index(idx)
    streamed = s.run(gpu.SeriesOptions(plain=True), z_host=z)
    assert np.array_equal(streamed["images"], resident["images"])


def test_fully_sampled_phantoms_are_recovered(gpu, ref):
    # test_nlinv.cpp:407-429 (default plan: M = 6, cg_tol 1e-3, max 200)
    N = 32
    for J in (1, 4):
        plan = gpu.make_plan(N, J)
        samples, angles = ref.phantom_series(J, 1, 51, 1, N, 0.0, 5)
        z = ref.grid_adjoint(plan, samples[0], angles[0])[None]
        P = ref.build_psf(plan, angles[0], 2 * N)[None]
        out = _run(gpu, plan, z, P, [0], gpu.SeriesOptions(plain=True))
        truth = ref.bandlimited_truth_rss(J, 5, 0, N)
        assert ref.nrmse_scaled(out["images"][0], truth) <= 0.05, J


def test_chaining_beats_scratch(gpu, ref):
    # test_nlinv.cpp:431-458
    N, F = 24, 12
    plan = _small_plan(gpu, N, 3, 6, 30)
    samples, angles = ref.phantom_series(3, F, 11, 5, N, 1e-3, 9)
    z = np.stack([ref.grid_adjoint(plan, samples[n], angles[n]) for n in range(F)])
    P = np.stack([ref.build_psf(plan, angles[n], 2 * N) for n in range(5)])
    idx = [n % 5 for n in range(F)]
    ch = _run(gpu, plan, z, P, idx, gpu.SeriesOptions(plain=True))
    sc = _run(gpu, plan, z, P, idx, gpu.SeriesOptions(plain=True, chain=False))
    wins = 0
    for n in range(6, F):
        truth = ref.bandlimited_truth_rss(3, 9, n, N)
        e_ch = ref.nrmse_scaled(ch["images"][n], truth)
        e_sc = ref.nrmse_scaled(sc["images"][n], truth)
        assert e_ch < 0.5
        wins += e_ch <= e_sc
    assert wins >= 5


def test_failing_frame_poisons_the_series(gpu, ref):
    # test_decomp.cpp:389-398
    plan = _small_plan(gpu, 16, 2, 2, 4)
    _, _, z, P, idx = _series_inputs(ref, plan, F=4, K=5, U=2)
    z[2, 0, 24, 24] = np.nan
    with pytest.raises(RuntimeError):
        _run(gpu, plan, z, P, idx, gpu.SeriesOptions(T=2, sched=gpu.TemporalSchedule(1, 1)))


def test_c1_series_against_reference(gpu, ref):
    # configs[0]: 64x64, G 128, 8 channels, 13 spokes, 5 frames, 7 Newton steps
    plan = gpu.raw_plan(128, 8)
    plan.newton_steps, plan.cg_iter_budget = 7, 50
    samples, angles, z, P, idx = _series_inputs(ref, plan, F=5, K=13, U=5, noise=0.0, seed=1234)
    want = ref.reconstruct_series(plan, samples, angles, plain=True)
    got = _run(gpu, plan, z, P, idx, gpu.SeriesOptions(plain=True))
    for n in range(5):
        assert rel_err(got["images"][n], want["images"][n]) < FRAME_TOL, n


def test_multi_device_series_matches_single_device(gpu, ref):
    # temporal decomposition across devices: with one visible GPU the device list
    # [0, 0] still exercises the peer-copy code path (UVA copies, worker devices);
    # with two or more GPUs the workers really run on different devices
    n = gpu.load_library().rtn_device_count()
    devices = [0, 1] if n >= 2 else [0, 0]
    plan = _small_plan(gpu, 16, 3, 3, 6)
    _, _, z, P, idx = _series_inputs(ref, plan, F=8, K=5, U=3)
    single = _run(gpu, plan, z, P, idx, gpu.SeriesOptions(T=1, sched=gpu.TemporalSchedule(2, 2)))
    ctx = gpu.Context(plan)
    s = gpu.Series(ctx, 8, P.shape[0], devices=devices)
    s.upload_frames(z)
    for k in range(P.shape[0]):
        s.upload_psf(k, P[k])
    s.set_psf_index(idx)
    out = s.run(gpu.SeriesOptions(T=1, sched=gpu.TemporalSchedule(2, 2)))
    # T = 1 over the device list: identical schedule, identical numerics
    assert np.array_equal(out["images"], single["images"])
    multi = s.run(gpu.SeriesOptions(T=2, sched=gpu.TemporalSchedule(2, 2)))
    for n_ in range(8):
        a = multi["audit"][n_]
        assert a.reg_final_src == n_ - 1 if n_ > 0 else a.init_src == -1
        assert np.sum(np.abs(multi["images"][n_]) ** 2) > 0


def test_c2_compressed_frame_against_reference(gpu, ref):
    # configs[1]: 160x160 image on a 320x320 grid (radix-5 line FFTs), 32 physical
    # channels PCA-compressed to 10 by the reference's calibrate_compression on the
    # first frames (rtnlinv_main.cpp:125-130), 15 spokes, 7 Newton steps
    plan = gpu.raw_plan(320, 10)
    plan.newton_steps, plan.cg_iter_budget = 7, 50
    samples, angles = ref.phantom_series(32, 2, 15, 5, plan.N, 1e-3, 1234)
    comp, energy = ref.compress_series(samples, angles, 10, 2)
    assert energy > 0.9
    z = ref.grid_adjoint(plan, comp[1], angles[1])
    P = ref.build_psf(plan, angles[1], 2 * plan.N)
    nsq = float(np.sum(np.abs(z.astype(np.complex128)) ** 2))
    z = (z * np.float32(100.0 / np.sqrt(nsq))).astype(np.complex64)
    init = gpu.initial_estimate(plan)
    with gpu.Context(plan) as ctx:
        ctx.set_psf(P)
        ctx.set_data(z)
        fr = ctx.reconstruct_frame(init)
    img, est, per, _ = ref.reconstruct_frame(plan, z, P, init, A=4)
    assert fr.cg_per_step == per
    assert rel_err(fr.image, img) < FRAME_TOL
    assert rel_err(fr.est, est) < FRAME_TOL


def _raw_series(gpu, plan, F, U, samples, angles, opts, cmat=None):
    ctx = gpu.Context(plan)
    s = gpu.Series(ctx, F, U)
    out = s.run(opts, raw=dict(samples=samples, angles=angles, cmat=cmat))
    out["series"], out["ctx"] = s, ctx
    return out


def test_raw_acquisitions_through_the_device_pre_stage(gpu, ref):
    # the reference's series driver grids and builds PSFs on the CPU (prep_series,
    # nlinv.cpp:366-402); here raw samples go H2D and the pre stage runs on the device
    plan = gpu.make_plan(24, 3)
    plan.newton_steps, plan.cg_iter_budget = 7, 30
    F, U = 7, 5
    samples, angles = ref.phantom_series(3, F, 11, U, plan.N, 1e-3, 23)
    want = ref.reconstruct_series(plan, samples, angles, plain=True)
    got = _raw_series(gpu, plan, F, U, samples, angles, gpu.SeriesOptions(plain=True))
    for n in range(F):
        assert rel_err(got["images"][n], want["images"][n]) < FRAME_TOL, n
    assert list(got["cg_iters"]) == list(want["cg_iters"])
    assert got["series"].psf_cache_size() == U  # PsfCache: one kernel per angle set
    # scheduled threads over the same raw input replay exactly like the gridded path
    sched = got["series"].run(gpu.SeriesOptions(T=2, sched=gpu.TemporalSchedule(2, 2)),
                              raw=dict(samples=samples, angles=angles))
    assert sched["audit"][F - 1].reg_final_src == F - 2


def test_raw_acquisitions_with_device_coil_compression(gpu, ref):
    # configs[1] style: physical channels PCA-compressed (calibrate_compression on the
    # first frames, rtnlinv_main.cpp:125-130), compression applied on the device
    plan = gpu.make_plan(24, 4)
    plan.newton_steps, plan.cg_iter_budget = 7, 30
    F, U, Jp = 5, 5, 12
    samples, angles = ref.phantom_series(Jp, F, 11, U, plan.N, 1e-3, 29)
    m, energy = ref.calibrate_compression(samples[:2], angles[:2], plan.J)
    comp, _ = ref.compress_series(samples, angles, plan.J, 2)
    want = ref.reconstruct_series(plan, comp, angles, plain=True)
    got = _raw_series(gpu, plan, F, U, samples, angles, gpu.SeriesOptions(plain=True), cmat=m)
    for n in range(F):
        assert rel_err(got["images"][n], want["images"][n]) < FRAME_TOL, n


@pytest.mark.parametrize("T,cluster", [(1, -1), (2, 1), (2, 0)])
def test_g256_series_cluster_and_pass_paths_match_reference(gpu, ref, T, cluster):
    # G = 256 instantiates the cluster-fused application (latency mode, on by default for
    # T = 1); both paths replay the reference frame by frame
    plan = gpu.raw_plan(256, 4)
    plan.newton_steps, plan.cg_iter_budget = 3, 9
    F = 4
    _, _, z, P, idx = _series_inputs(ref, plan, F=F, K=15, U=2, noise=0.0, seed=4)
    out = _run(gpu, plan, z, P, idx, gpu.SeriesOptions(T=T, plain=(T == 1), cluster=cluster,
                                                       sched=gpu.TemporalSchedule(1, 1)))
    M = plan.newton_steps
    scale = out["series"].normalize()
    zs = (z * np.float32(scale)).astype(np.complex64)
    unity = gpu.initial_estimate(plan)
    ests = {}
    for n in range(F):
        a = out["audit"][n]
        init = unity if a.init_src < 0 else ests[a.init_src]
        regs = [unity if a.init_src < 0 else ests[a.reg_src[m]] for m in range(M)]
        img, est, _ = ref.reconstruct_frame_regs(plan, zs[n], P[idx[n]], init, regs)
        ests[n] = est
        assert rel_err(out["images"][n], img * np.float32(1.0 / scale)) < FRAME_TOL, n


def test_psf_cache_sidecar_interchanges_with_the_reference(gpu, ref, tmp_path):
    # PsfCache::save / load (preproc.cpp:346-388): the device cache writes and reads the
    # reference's "PSFC" v1 file
    plan = gpu.make_plan(24, 3)
    plan.newton_steps, plan.cg_iter_budget = 3, 9
    F, U = 5, 5
    samples, angles = ref.phantom_series(3, F, 11, U, plan.N, 1e-3, 41)
    s = gpu.Series(gpu.Context(plan), F, U)
    s.run(gpu.SeriesOptions(plain=True), raw=dict(samples=samples, angles=angles))
    ours = tmp_path / "ours.psfc"
    s.save_psf_cache(ours)
    for n in range(U):  # the reference loads our file and finds every kernel (no rebuild)
        P, hits, size = ref.psf_cache_get(plan, ours, angles[n], 2 * plan.N)
        assert hits == 1 and size == U
        assert rel_err(P, ref.build_psf(plan, angles[n], 2 * plan.N)) < 1e-5
    theirs = tmp_path / "theirs.psfc"
    ref.psf_cache_save(plan, angles[:U], 2 * plan.N, theirs)
    s2 = gpu.Series(gpu.Context(plan), F, U)
    s2.load_psf_cache(theirs)
    assert s2.psf_cache_size() == U
    out = s2.run(gpu.SeriesOptions(plain=True), raw=dict(samples=samples, angles=angles))
    assert s2.psf_cache_size() == U  # every angle set hit the loaded cache
    want = ref.reconstruct_series(plan, samples, angles, plain=True)
    for n in range(F):
        assert rel_err(out["images"][n], want["images"][n]) < FRAME_TOL, n
    (tmp_path / "bad.psfc").write_bytes(b"nope")
    with pytest.raises(gpu.DataError):
        s2.load_psf_cache(tmp_path / "bad.psfc")


@pytest.mark.parametrize("T", [2, 3])
def test_zero_rhs_frames_recover_through_the_safe_mode_rerun(gpu, ref, T):
    """a speculative budget split that meets an exactly-zero right-hand side
    (frame_verify fails) while other workers wait on the poisoned ledgers must end in the
    safe-mode re-run, not in a spurious DecompFault. All-zero frames chained from the
    initial estimate give zero rhs in every step (nlinv.cpp:182-186: 0 iterations)."""
    plan = _small_plan(gpu, 16, 2, 3, 9)
    F = 6
    samples = np.zeros((F, plan.J, 5, 2 * plan.N), np.complex64)
    _, angles = ref.phantom_series(plan.J, F, 5, 3, plan.N, 0.0, 3)
    z = np.zeros((F, plan.J, plan.G, plan.G), np.complex64)
    P = np.stack([ref.build_psf(plan, angles[n], 2 * plan.N) for n in range(3)])
    out = _run(gpu, plan, z, P, [n % 3 for n in range(F)],
               gpu.SeriesOptions(T=T, sched=gpu.TemporalSchedule(1, 1)))
    want = ref.reconstruct_series(plan, samples, angles, T=1, sched=(1, 1))
    assert list(out["cg_iters"]) == list(want["cg_iters"]) == [0] * F
    assert np.array_equal(out["images"], want["images"])
    for n in range(1, F):
        assert out["audit"][n].reg_final_src == n - 1


@pytest.mark.parametrize("mode", ["magnitude", "median3", "phase_difference"])
def test_series_images_through_the_device_post_stage_into_an_rti_sink(gpu, ref, tmp_path, mode):
    """device postprocessing of the series images straight into the
    .rti sink; the reference's RtiReader reads the file and the pixels match the
    reference's own postprocessing of the reference's images (pipeline.cpp:60-137)"""
    plan = _small_plan(gpu, 24, 3, 3, 9)
    F = 6
    samples, angles = ref.phantom_series(3, F, 11, 5, plan.N, 1e-3, 19)
    want = ref.reconstruct_series(plan, samples, angles, plain=True)
    s = gpu.Series(gpu.Context(plan), F, 5)
    s.run(gpu.SeriesOptions(plain=True), raw=dict(samples=samples, angles=angles))
    header = [1, plan.N, 3, 11, 5, F, 2, 2 if mode == "phase_difference" else 1, 2 * plan.N]
    path = tmp_path / "out.rti"
    with gpu.RtiSink(path, header) as sink:
        s.write_rti(sink, 0, F, mode=mode, slice_id=1)
    h, recs, px = ref.rti_read(path)
    assert h == header
    if mode == "phase_difference":
        assert recs == [(k, 1, 1) for k in range(F // 2)]
        expect = np.stack([ref.phase_difference_image(want["images"][2 * k], want["images"][2 * k + 1])
                           for k in range(F // 2)])
        # phases: compare on the unit circle where the magnitude is meaningful
        mag = np.abs(want["images"][0::2]) * np.abs(want["images"][1::2])
        keep = mag > 1e-3 * mag.max()
        assert np.max(np.abs(np.angle(np.exp(1j * (px - expect)))[keep])) < 1e-2
    else:
        assert recs == [(n, 1, 0) for n in range(F)]
        mags = np.stack([ref.magnitude_image(want["images"][n]) for n in range(F)])
        expect = ref.median_filter(mags) if mode == "median3" else mags
        assert rel_err(px, expect) < FRAME_TOL


def _slice_inputs(ref, plan, Sl, F, K, U, seeds):
    """Sl slices of F frames each (a different phantom seed per slice), interleaved in
    the pipeline's delivery order g = frame * Sl + slice"""
    per = [ref.phantom_series(plan.J, F, K, U, plan.N, 1e-4, seeds[sl]) for sl in range(Sl)]
    samples = np.stack([per[g % Sl][0][g // Sl] for g in range(F * Sl)])
    angles = np.stack([per[g % Sl][1][g // Sl] for g in range(F * Sl)])
    return per, samples, angles


def test_interleaved_slices_equal_independent_series_bit_for_bit(gpu, ref):
    """per-slice chains in one device series (pipeline.cpp:315-334).
    Each slice is its own chain with its own normalisation, so a 2-slice interleaved
    series reproduces two separate single-slice series bit for bit, and each slice
    matches the reference's own series on that slice's frames."""
    plan = _small_plan(gpu, 24, 3, 3, 9)
    Sl, F, U = 2, 5, 5
    per, samples, angles = _slice_inputs(ref, plan, Sl, F, 11, U, [21, 22])
    s = gpu.Series(gpu.Context(plan), F * Sl, F * Sl)
    s.set_slices(Sl)
    out = s.run(gpu.SeriesOptions(plain=True), raw=dict(samples=samples, angles=angles))
    for sl in range(Sl):
        single = gpu.Series(gpu.Context(plan), F, U)
        alone = single.run(gpu.SeriesOptions(plain=True), raw=dict(samples=per[sl][0], angles=per[sl][1]))
        got = out["images"][sl::Sl]
        assert np.array_equal(got, alone["images"]), sl
        assert s.slice_scale(sl) == single.normalize()
        want = ref.reconstruct_series(plan, per[sl][0], per[sl][1], plain=True)
        assert want["data_scale"] == pytest.approx(s.slice_scale(sl), rel=1e-6)
        for n in range(F):
            assert rel_err(got[n], want["images"][n]) < FRAME_TOL, (sl, n)
    assert [a.frame for a in out["audit"]] == [g // Sl for g in range(F * Sl)]


@pytest.mark.parametrize("lanes", ["0", "1"])
def test_interleaved_slices_with_frames_in_flight_replay_per_slice(gpu, ref, lanes, monkeypatch):
    """T = 3 workers over 2 interleaved slices with a short strict prefix: every slice
    keeps the ordering contract on its own chain and replays through the reference.
    lanes = 1: workers 1 and 2 run the pre stage of their own frames (RTN_PRE_LANES, the
    multi-GPU layout) and normalise the slices whose first frame they receive"""
    monkeypatch.setenv("RTN_PRE_LANES", lanes)
    plan = _small_plan(gpu, 16, 3, 3, 6)
    Sl, F, U = 2, 6, 3
    per, samples, angles = _slice_inputs(ref, plan, Sl, F, 5, U, [31, 32])
    sched = gpu.TemporalSchedule(2, 2)
    s = gpu.Series(gpu.Context(plan), F * Sl, F * Sl)
    s.set_slices(Sl)
    out = s.run(gpu.SeriesOptions(T=3, sched=sched), raw=dict(samples=samples, angles=angles))
    M = plan.newton_steps
    unity = gpu.initial_estimate(plan)
    for sl in range(Sl):
        audit = out["audit"][sl::Sl]
        z = np.stack([ref.grid_adjoint(plan, per[sl][0][n], per[sl][1][n]) for n in range(F)])
        P = np.stack([ref.build_psf(plan, per[sl][1][n], 2 * plan.N) for n in range(F)])
        scale = s.slice_scale(sl)
        zs = (z * np.float32(scale)).astype(np.complex64)
        ests = {}
        for n in range(F):
            a = audit[n]
            assert a.frame == n
            if n > 0:
                assert 0 <= a.init_src < n and a.reg_final_src == n - 1
                assert a.reg_final_seq > audit[n - 1].finish_seq
                if n <= sched.l:
                    assert a.start_seq > audit[n - 1].finish_seq
            init = unity if a.init_src < 0 else ests[a.init_src]
            regs = [unity if a.init_src < 0 else ests[a.reg_src[m]] for m in range(M)]
            img, est, _ = ref.reconstruct_frame_regs(plan, zs[n], P[n], init, regs)
            ests[n] = est
            assert rel_err(out["images"][n * Sl + sl], img * np.float32(1.0 / scale)) < FRAME_TOL, (sl, n)
            assert rel_err(s.estimate(n * Sl + sl), est) < FRAME_TOL, (sl, n)


def test_pre_stage_lanes_equal_the_store_path(gpu, ref, monkeypatch):
    # the raw-input pre stage on per-worker lanes (own stream, Preproc, staging, PSF cache,
    # gridded frames; the multi-GPU layout, forced on one GPU) against the store's single
    # copy stream: with compression, T = 3 workers and a fully sequential schedule the
    # frames are bit-identical
    plan = gpu.make_plan(24, 4)
    plan.newton_steps, plan.cg_iter_budget = 5, 20
    F, U, Jp = 7, 3, 8
    samples, angles = ref.phantom_series(Jp, F, 11, U, plan.N, 1e-3, 37)
    m, _ = ref.calibrate_compression(samples[:2], angles[:2], plan.J)
    outs = {}
    for lanes in ("0", "1"):
        monkeypatch.setenv("RTN_PRE_LANES", lanes)
        s = gpu.Series(gpu.Context(plan), F, U)
        outs[lanes] = s.run(gpu.SeriesOptions(T=3, sched=gpu.TemporalSchedule(F, 1)),
                            raw=dict(samples=samples, angles=angles, cmat=m))
        outs[lanes]["scale"] = s.slice_scale(0)
    assert list(outs["0"]["cg_iters"]) == list(outs["1"]["cg_iters"])
    assert outs["0"]["scale"] == outs["1"]["scale"]
    for n in range(F):
        assert np.array_equal(outs["0"]["images"][n], outs["1"]["images"][n]), n
