"""Solver seams on the GPU vs the CPU oracle (reference solver.py:141-306, model.py:133-152)."""
import numpy as np
import pytest

import oracle.ringflow_np as O
import scenarios

pytestmark = pytest.mark.gpu
T, D = 32, 4
SHAPE = (T, D)


@pytest.fixture(scope="module")
def rf():
    import paper_2605_28657_b200 as m

    return m


def rnd(tag, seed=17):
    return scenarios.keyed(seed, tag, SHAPE)


def test_sde_bit_exact(rf):
    x, v, src = rnd("x"), rnd("v"), rnd("src")
    curve = O.uniform(8, 0, 0, "curve", (T,))
    for step, (tc, tn) in enumerate([(1.0, 0.7), (0.7, 0.3), (0.3, 0.0)]):
        got = rf.sde_step(x, v, tc, tn, src, rf.make_curves(T, sde_denoise_curve=curve),
                          rf.StepState(8, step), rf.NoiseSource(23, 6))
        want = O.sde(x, v, tc, tn, src, {"sde_denoise_curve": curve}, O.State(8), 23, 6) if step == 0 else None
        st = O.State(8)
        st.step = step
        want = O.sde(x, v, tc, tn, src, {"sde_denoise_curve": curve}, st, 23, 6)
        assert np.array_equal(got, want)


def test_sde_identities(rf):
    x, v, src = rnd("x"), rnd("v"), rnd("src")
    rng = rf.NoiseSource(23, 6)
    got = rf.sde_step(x, v, 1.0, 0.4, src, rf.make_curves(T, sde_denoise_curve=1.0), rf.StepState(8), rng)
    noise = rng.normal(0, "sde", SHAPE)
    assert np.max(np.abs(got - (0.4 * noise + 0.6 * (x - v)))) <= 1e-12
    # curve == 0 lands on the source bit-exactly over a full schedule (C11(b))
    model = rf.ToyFlowModel(T, D)
    w = rf.ModelWeights.zeros(SHAPE)
    cond = rf.ConditionSet(prompt_hash=rf.prompt_id("identity"))
    sched = rf.build_schedule(1.0, 8)
    zero = rf.make_curves(T, sde_denoise_curve=0.0)
    xt = rng.normal(0, "init", SHAPE)
    for k in range(8):
        vel = model.velocity(xt, sched.sigmas[k], cond, w, rng, k)
        xt = rf.sde_step(xt, vel, sched.sigmas[k], sched.sigmas[k + 1], src, zero, rf.StepState(8, k), rng)
    assert np.array_equal(xt, src)
    with pytest.raises(rf.MissingSourceError):
        rf.sde_step(x, v, 1.0, 0.5, None, rf.make_curves(T, sde_denoise_curve=0.5), rf.StepState(8), rng)
    with pytest.raises(ValueError):
        rf.sde_step(x, v, 0.5, 0.5, src, rf.CurveSet(), rf.StepState(8), rng)


def test_morph_and_sentinels(rf):
    x, v, src, tgt = rnd("x"), rnd("v"), rnd("src"), rnd("target")
    rng = rf.NoiseSource(23, 6)
    bare = rf.sde_step(x, v, 0.5, 0.2, src, rf.CurveSet(x0_target=tgt), rf.StepState(8, 4), rng)
    dressed = rf.sde_step(x, v, 0.5, 0.2, src, rf.make_curves(T, x0_target=tgt, sde_denoise_curve=1.0,
                                                               x0_target_strength=1.0), rf.StepState(8, 4), rng)
    assert np.array_equal(bare, dressed)
    st = O.State(8)
    st.step = 4
    assert np.array_equal(bare, O.sde(x, v, 0.5, 0.2, src, {"x0_target": tgt}, st, 23, 6))
    early = rf.sde_step(x, v, 0.5, 0.2, src, rf.CurveSet(x0_target=tgt), rf.StepState(8, 3), rng)
    st.step = 3
    assert np.array_equal(early, O.sde(x, v, 0.5, 0.2, src, {}, st, 23, 6))


def test_ode_bit_exact(rf):
    x, v, tgt = rnd("x"), rnd("v"), rnd("target")
    rng = rf.NoiseSource(3, 4)
    vs = np.linspace(0.2, 1.5, T)
    for step in (2, 5):
        cv = rf.make_curves(T, velocity_scale=vs, ode_noise_curve=0.25, x0_target=tgt,
                            x0_target_strength=np.linspace(0, 1, T))
        got = rf.ode_step(x, v, 0.6, 0.35, cv, rng, rf.StepState(8, step))
        st = O.State(8)
        st.step = step
        want = O.ode(x, v, 0.6, 0.35, {"velocity_scale": cv.velocity_scale, "ode_noise_curve": cv.ode_noise_curve,
                                        "x0_target": tgt, "x0_target_strength": cv.x0_target_strength}, st, 3, 4)
        assert np.array_equal(got, want)
    plain = rf.ode_step(x, v, 1.0, 0.5, rf.CurveSet(), rng)
    assert np.array_equal(plain, x + v * (0.5 - 1.0))
    zero = rf.ode_step(x, v, 1.0, 0.5, rf.make_curves(T, velocity_scale=0.0), rng)
    assert np.array_equal(zero, x)


def test_toy_velocity_bit_exact(rf):
    model = rf.ToyFlowModel(T, D, perturbation=0.1)
    w = rf.ModelWeights.zeros(SHAPE)
    cond = rf.ConditionSet(prompt_hash=rf.prompt_id("v"), hint_strength=0.7, timbre_strength=0.3)
    x = rnd("x")
    got = model.velocity(x, 0.75, cond, w, rf.NoiseSource(5, 9), 3)
    toy = O.Toy(T, D, 0.1)
    want = toy.velocity(x, 0.75, O.Cond(rf.prompt_id("v"), 0.7, 0.3), np.zeros(SHAPE), 5, 9, 3)
    assert np.array_equal(got, want)
    assert np.array_equal(model.pattern("hint", 42), toy.pattern("hint", 42))
    assert np.array_equal(model.x0_of(cond, w), toy.x0(O.Cond(rf.prompt_id("v"), 0.7, 0.3), np.zeros(SHAPE)))
    with pytest.raises(ValueError):
        model.velocity(x, 0.0, cond, w, rf.NoiseSource(0), 0)


@pytest.mark.parametrize("mode", ["off", "full-cfg", "onetime-negative", "self-negative"])
def test_guided_velocity_modes(rf, mode):
    vc, vu = rnd("vc"), rnd("vu")
    st_gpu, st_cpu = rf.StepState(8), O.State(8)
    cv = rf.make_curves(T, guidance_enabled=True, rcfg_mode=mode, guidance_curve=np.linspace(1, 5, T),
                        apg_momentum=0.3)
    host = {"guidance_curve": cv.guidance_curve, "apg_momentum": cv.apg_momentum}
    for k in range(3):
        vck = vc * (1 + k)
        got = rf.guided_velocity(vck, vu, cv, st_gpu, k)
        want = O.guided(vck, vu, host, mode, st_cpu)
        assert np.array_equal(got, want), k
    # every mode at scale 1 equals guidance off (C11(d))
    out = rf.guided_velocity(vc, vu, rf.CurveSet(guidance_enabled=True, rcfg_mode=mode), rf.StepState(8), 0)
    assert np.array_equal(out, vc)


def test_guided_rescale_tolerance(rf):
    vc, vu = rnd("vc"), rnd("vu")
    cv = rf.make_curves(T, guidance_enabled=True, guidance_curve=3.0, cfg_rescale_curve=np.linspace(0, 1, T))
    got = rf.guided_velocity(vc, vu, cv, rf.StepState(8), 0)
    want = O.guided(vc, vu, {"guidance_curve": cv.guidance_curve, "cfg_rescale_curve": cv.cfg_rescale_curve},
                    "off", O.State(8))
    assert np.max(np.abs(got - want)) <= 1e-13 * max(1.0, np.max(np.abs(want)))


def test_blend_conditions(rf):
    vs = [rnd("a"), rnd("b"), rnd("c")]
    ws = [np.linspace(0, 1, T), np.ones(T), np.linspace(2, 0.5, T)]
    assert np.array_equal(rf.blend_conditions(vs, ws), O.blend(vs, ws))
    assert rf.blend_conditions(vs[:1], ws[:1]) is vs[0]
    with pytest.raises(ValueError):
        rf.blend_conditions(vs[:2], [np.zeros(T), np.zeros(T)])
    with pytest.raises(ValueError):
        rf.blend_conditions(vs[:2], [-np.ones(T), np.ones(T)])


def test_metrics(rf):
    a, b = rnd("a"), rnd("b")
    assert rf.mse(a, a) == 0.0
    assert abs(rf.mse(a, b) - O.mse(a, b)) <= 1e-15 * O.mse(a, b)
    assert rf.mse(np.zeros((4, 2)), np.ones((4, 2))) == 1.0
    assert rf.rms_diff(np.zeros((4, 2)), np.ones((4, 2))) == 1.0
    s = rf.segment_cosine_similarity(a, a, 4)
    assert np.allclose(s, 1.0)
    with pytest.raises(rf.ShapeMismatchError):
        rf.mse(a, b[:3])
