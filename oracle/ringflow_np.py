"""CPU oracle: a float64 numpy restatement of the reference hot path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline / reference arm may import this module; the product package
(paper_2605_28657_b200/) never does.  It restates, in one self-contained module, the
reference's per-tick path so GPU results can be checked on arbitrary seeded inputs and
so the reference's CPU cost can be timed on the GPU box (where /root/reference does
not exist).  Each piece cites the reference function it restates
(paths relative to /root/reference/pkg/src/ringflow/).

Pinning: tests/test_oracle.py checks this module against golden vectors produced by
running the real reference in the build container (tests/golden/make_goldens.py):
bit-exact latents, records, schedules and PCM for every committed scenario.

Noise is drawn exactly as the reference does (numpy Philox4x64-10 + ziggurat via
np.random.Generator), i.e. through the third-party dependency itself (numpy 2.3.5 in
this image); oracle/npyrandom.c restates that algorithm in C and is pinned against
numpy separately.
"""
from __future__ import annotations

import hashlib
import math
import struct
from collections import deque

import numpy as np

# ------------------------------------------------------------------ latents.py ----


def feed(h, part):  # latents.py:80-101
    if isinstance(part, bool):
        part = int(part)
    if isinstance(part, int):
        h.update(b"i" + part.to_bytes(16, "little", signed=True))
    elif isinstance(part, float):
        h.update(b"f" + struct.pack("<d", part))
    elif isinstance(part, str):
        h.update(b"s" + part.encode("utf-8"))
    elif isinstance(part, bytes):
        h.update(b"b" + part)
    elif isinstance(part, np.ndarray):
        h.update(b"a" + str(part.shape).encode() + np.ascontiguousarray(part, dtype=np.float64).tobytes())
    elif part is None:
        h.update(b"n")
    elif isinstance(part, (tuple, list)):
        h.update(b"(")
        for p in part:
            feed(h, p)
        h.update(b")")
    else:
        raise TypeError(type(part))


def chash(*parts) -> int:  # latents.py:104-109
    h = hashlib.blake2b(digest_size=8)
    for p in parts:
        feed(h, p)
    return int.from_bytes(h.digest(), "little") & (2**63 - 1)


def prompt_id(text):  # latents.py:112-114
    return chash("prompt", text)


def philox_key(seed, stream, step, tag) -> int:  # latents.py:130-135
    h = hashlib.blake2b(digest_size=16)
    h.update(struct.pack("<qq", seed, step))
    h.update(stream.to_bytes(16, "little", signed=True))
    h.update(tag.encode("utf-8"))
    return int.from_bytes(h.digest(), "little")


def normal(seed, stream, step, tag, shape):  # latents.py:144-146
    return np.random.Generator(np.random.Philox(key=philox_key(seed, stream, step, tag))).standard_normal(shape)


def uniform(seed, stream, step, tag, shape):  # latents.py:148-150
    return np.random.Generator(np.random.Philox(key=philox_key(seed, stream, step, tag))).random(shape)


def mse(a, b):  # latents.py:42-46
    d = a - b
    return float(np.mean(d * d))


# ------------------------------------------------------------------ schedule.py ---


def sigmas_of(denoise, steps, shift):  # schedule.py:43-64
    u = 1.0 - np.arange(steps + 1, dtype=np.float64) / steps
    s = denoise * (shift * u / (1.0 + (shift - 1.0) * u))
    s[0] = denoise
    s[-1] = 0.0
    return s


def schedule_id(sig, shift):  # schedule.py:66-68
    h = hashlib.blake2b(digest_size=6)
    h.update(sig.tobytes())
    h.update(np.float64(shift).tobytes())
    return h.hexdigest()


class Sched:
    def __init__(self, denoise, steps, shift):
        self.denoise, self.steps, self.shift = denoise, steps, shift
        self.sigmas = sigmas_of(denoise, steps, shift)
        self.schedule_id = schedule_id(self.sigmas, shift)


class SchedCache:  # schedule.py:78-95
    def __init__(self):
        self.d = {}

    def get(self, denoise, steps, shift):
        k = (round(denoise / 1e-6), steps, shift)
        if k not in self.d:
            self.d[k] = Sched(denoise, steps, shift)
        return self.d[k]


# --------------------------------------------------------------------- model.py ---

MULT = {"sde_denoise_curve", "guidance_curve", "velocity_scale", "cfg_rescale_curve", "x0_target_strength"}
RANGES = {"sde_denoise_curve": (0.0, 1.0), "guidance_curve": (0.0, 8.0), "velocity_scale": (0.0, 4.0),
          "ode_noise_curve": (0.0, 1.0), "apg_momentum": (-1.0, 1.0), "cfg_rescale_curve": (0.0, 1.0),
          "x0_target_strength": (0.0, 1.0)}
FIELDS = tuple(RANGES)


def clamp(name, values, frames):  # solver.py:71-83
    lo, hi = RANGES[name]
    arr = np.asarray(values, dtype=np.float64)
    if arr.ndim == 0:
        arr = np.full(frames, float(arr))
    return np.clip(arr, lo, hi)


class Cond:
    """ConditionSet (model.py:33-64) as a plain record."""

    def __init__(self, prompt_hash, hint=0.0, timbre=0.0, source=None, weight=None):
        self.prompt_hash, self.hint, self.timbre, self.source, self.weight = prompt_hash, hint, timbre, source, weight

    def content_key(self):
        return chash(self.prompt_hash, self.hint, self.timbre, self.source, self.weight)


class Request:
    """GenerationRequest (pipeline.py:77-96); curves: dict name -> array, plus flags."""

    def __init__(self, conds, curves=None, solver="sde", x0_target=None, guidance=False, rcfg="off"):
        self.conds, self.solver = tuple(conds), solver
        self.curves = dict(curves or {})
        self.x0_target, self.guidance, self.rcfg = x0_target, guidance, rcfg

    @property
    def source(self):
        return self.conds[0].source

    def content_key(self):
        return chash([c.content_key() for c in self.conds], self.solver)


class Toy:
    """ToyFlowModel (model.py:91-152)."""

    def __init__(self, frames, channels, jitter):
        self.T, self.D, self.jitter = frames, channels, jitter
        self.cache = {}

    def pattern(self, kind, ph):  # model.py:104-121
        key = (kind, ph)
        if key not in self.cache:
            stream = chash("pattern", kind)
            amps = normal(ph, stream, 0, "amps", (4, self.D))
            phases = 2.0 * np.pi * uniform(ph, stream, 0, "phases", (4, self.D))
            t = (np.arange(self.T, dtype=np.float64) + 0.5) / self.T
            out = np.zeros((self.T, self.D))
            for k in range(4):
                out += amps[k][None, :] * np.sin(2.0 * np.pi * (k + 1) * t[:, None] + phases[k][None, :])
            out /= np.sqrt(4)
            self.cache[key] = out
        return self.cache[key]

    def x0(self, c, style):  # model.py:123-131
        x0 = self.pattern("base", c.prompt_hash).copy()
        if c.hint != 0.0:
            x0 += c.hint * 0.45 * self.pattern("hint", c.prompt_hash)
        if c.timbre != 0.0:
            x0 += c.timbre * 0.45 * self.pattern("timbre", c.prompt_hash)
        x0 += style
        return x0

    def velocity(self, x, t, c, style, seed, stream, step):  # model.py:133-152
        v = (x - self.x0(c, style)) / t
        if self.jitter != 0.0:
            v = v + self.jitter * t * normal(seed, stream, step, "model", x.shape)
        return v


# -------------------------------------------------------------------- solver.py ---


class State:  # solver.py:118-134
    def __init__(self, total):
        self.total, self.step = total, 0
        self.momentum = self.residual = self.prev = None

    def refine(self):
        return self.step >= self.total // 2


def guided(vc, vu, curves, rcfg, st):  # solver.py:141-201
    if rcfg in ("off", "full-cfg"):
        neg = vu
    elif rcfg == "onetime-negative":
        if st.residual is None:
            st.residual = vc - vu
        neg = vc - st.residual
    else:
        neg = vu if st.prev is None else st.prev
        st.prev = vc.copy()
    delta = vc - neg
    apg = curves.get("apg_momentum")
    if apg is not None:
        if st.momentum is None:
            st.momentum = np.zeros_like(vc)
        st.momentum = apg[:, None] * st.momentum + delta
        delta = st.momentum
    scale = curves.get("guidance_curve")
    if scale is None:
        scale = np.ones(vc.shape[0])
    out = vc + (scale - 1.0)[:, None] * delta
    keep = curves.get("cfg_rescale_curve")
    if keep is not None:
        no = np.linalg.norm(out, axis=1)
        npos = np.linalg.norm(vc, axis=1)
        bl = keep * no + (1.0 - keep) * npos
        out = out * np.where(no > 0.0, bl / np.where(no > 0.0, no, 1.0), 1.0)[:, None]
    return out


def blend(vs, ws):  # solver.py:204-227
    if len(vs) == 1:
        return vs[0]
    tot = np.zeros_like(ws[0])
    acc = np.zeros_like(vs[0])
    for v, w in zip(vs, ws):
        acc += w[:, None] * v
        tot += w
    return acc / tot[:, None]


def morph(x0p, curves, st):  # solver.py:230-238
    tgt = curves.get("x0_target")
    if tgt is None or not st.refine():
        return x0p
    s = curves.get("x0_target_strength")
    a = (np.ones(x0p.shape[0]) if s is None else s)[:, None]
    return (1.0 - a) * x0p + a * tgt


def sde(x, v, tc, tn, source, curves, st, seed, stream):  # solver.py:273-306
    x0p = morph(x - v * tc, curves, st)
    n = normal(seed, stream, st.step, "sde", x.shape)
    full = tn * n + (1.0 - tn) * x0p
    c = curves.get("sde_denoise_curve")
    if source is None:
        if c is not None and np.any(c < 1.0):
            raise ValueError("MissingSource")
        return full
    if c is None:
        c = np.ones(x.shape[0])
    srcp = tn * n + (1.0 - tn) * source
    return c[:, None] * full + (1.0 - c[:, None]) * srcp


def ode(x, v, tc, tn, curves, st, seed, stream):  # solver.py:241-270
    if st is not None and curves.get("x0_target") is not None and st.refine():
        v = (x - morph(x - v * tc, curves, st)) / tc
    vs = curves.get("velocity_scale")
    if vs is not None:
        v = vs[:, None] * v
    xn = x + v * (tn - tc)
    on = curves.get("ode_noise_curve")
    if on is not None:
        xn = xn + on[:, None] * normal(seed, stream, 0 if st is None else st.step, "ode", x.shape)
    return xn


# ------------------------------------------------------------------ pipeline.py ---


class Record:
    def __init__(self, **kw):
        self.__dict__.update(kw)


class Slot:
    def __init__(self, sid, req, denoise, sched, x, total, stream, tick):
        self.sid, self.req, self.denoise, self.sched, self.x = sid, req, denoise, sched, x
        self.st, self.stream, self.admitted = State(total), stream, tick
        self.ids, self.migrated = {sched.schedule_id}, False


class Pipeline:
    """StreamPipeline (pipeline.py:247-566) restated over plain records."""

    def __init__(self, depth=8, steps=8, frames=96, channels=8, mode="per-slot", threshold=1e-3, seed=0,
                 shift=3.0, denoise=1.0, jitter=0.1, auto_submit=True, request=None):
        self.depth, self.steps, self.T, self.D = depth, steps, frames, channels
        self.mode, self.threshold, self.seed, self.shift = mode, threshold, seed, shift
        self.denoise, self.auto = denoise, auto_submit
        self.model = Toy(frames, channels, jitter)
        self.style = np.zeros((frames, channels))
        self.cache = SchedCache()
        self.reg = {}
        self.template = request
        self.slots = [None] * depth
        self.queue = deque()
        self.tick_index = self.completions = self.submissions = 0
        self.prev_denoise = denoise
        self.reference = self.last = None
        self.spacing = math.ceil(steps / depth)
        self.warmup = depth
        self.last_admit = None
        self.refusals = 0
        self.last_timesteps = []

    # control (pipeline.py:306-345)
    def _mark(self):
        if self.last is not None:
            self.reference = self.last.copy()

    def set_request(self, r):
        self._mark()
        self.template = r

    def set_denoise(self, v):
        self._mark()
        self.denoise = float(v)

    def set_shared_curve(self, name, value):
        self._mark()
        self.reg[name] = np.asarray(value, dtype=np.float64) if name == "x0_target" else clamp(name, value, self.T)

    def set_model_weights(self, offset):
        self._mark()
        self.style = np.array(offset, dtype=np.float64)

    def set_mode(self, mode):
        self._mark()
        self.mode = mode
        self.prev_denoise = self.denoise

    def submit(self, req=None):  # pipeline.py:349-368
        if len(self.queue) >= self.depth:
            raise RuntimeError("backpressure")
        return self._enqueue(req)

    def _enqueue(self, req):
        req = req if req is not None else self.template
        if self.denoise < 1.0 and req.source is None:
            raise ValueError("denoise < 1 requires source")
        sub = (self.submissions, req, self.denoise, self.cache.get(self.denoise, self.steps, self.shift))
        self.submissions += 1
        self.queue.append(sub)
        return sub[0]

    def tick(self):  # pipeline.py:372-398
        if self.mode == "migration":
            tgt = self.cache.get(self.denoise, self.steps, self.shift)
            for s in self.slots:
                if s is None or s.sched.schedule_id == tgt.schedule_id:
                    continue
                if tgt.steps != s.sched.steps:
                    self.refusals += 1
                    continue
                s.sched, s.denoise, s.migrated = tgt, tgt.denoise, True
                s.ids.add(tgt.schedule_id)
        if self.mode == "global-reset" and self.denoise != self.prev_denoise:
            self.slots = [None] * self.depth
            self.warmup = self.depth
            self.last_admit = None
        active = [s for s in self.slots if s is not None]
        self.last_timesteps = [(s.sched.sigmas[s.st.step], s.sched.schedule_id) for s in active]
        for s in active:
            self._step(s)
        out = []
        for i, s in enumerate(self.slots):
            if s is not None and s.st.step >= self.steps:
                out.append(self._emit(s))
                self.slots[i] = None
        self._refill()
        self.prev_denoise = self.denoise
        self.tick_index += 1
        return out

    def snapshot(self):  # pipeline.py:289-304 (PipelineSnapshot / SlotView)
        from types import SimpleNamespace as NS

        slots = tuple(None if s is None else NS(denoise=s.denoise, step=s.st.step, schedule_id=s.sched.schedule_id)
                      for s in self.slots)
        return NS(slots=slots, queue_depth=len(self.queue), mode=self.mode, tick=self.tick_index,
                  denoise=self.denoise, denoise_values=lambda: {v.denoise for v in slots if v is not None})

    def curves_of(self, s):  # pipeline.py:415-422
        c = dict(s.req.curves)
        c["x0_target"] = s.req.x0_target
        c.update(self.reg)
        if c.get("x0_target") is None:
            c.pop("x0_target_strength", None)
        return c

    def _step(self, s):  # pipeline.py:424-464
        k = s.st.step
        tc, tn = float(s.sched.sigmas[k]), float(s.sched.sigmas[k + 1])
        curves = self.curves_of(s)
        vs = [self.model.velocity(s.x, tc, c, self.style, self.seed, s.stream, k) for c in s.req.conds]
        if len(vs) == 1:
            v = vs[0]
        else:
            v = blend(vs, [c.weight if c.weight is not None else np.ones(self.T) for c in s.req.conds])
        if s.req.guidance:
            need = (s.req.rcfg in ("off", "full-cfg") or (s.req.rcfg == "onetime-negative" and s.st.residual is None)
                    or (s.req.rcfg == "self-negative" and s.st.prev is None))
            vu = self.model.velocity(s.x, tc, Cond(0), self.style, self.seed, s.stream, k) if need else None
            v = guided(v, vu, curves, s.req.rcfg, s.st)
        if s.req.solver == "sde":
            s.x = sde(s.x, v, tc, tn, s.req.source, curves, s.st, self.seed, s.stream)
        else:
            s.x = ode(s.x, v, tc, tn, curves, s.st, self.seed, s.stream)
        s.st.step += 1
        s.ids.add(s.sched.schedule_id)

    def _emit(self, s):  # pipeline.py:466-491
        lat = s.x.copy()
        if not np.all(np.isfinite(lat)):
            raise RuntimeError("non-finite")
        hybrid = len(s.ids) > 1
        skipped = self.last is not None and mse(lat, self.last) < self.threshold
        rms = float(np.sqrt(mse(lat, self.reference))) if self.reference is not None else None
        rec = Record(latent=lat, tick=self.tick_index, completion_index=self.completions, submission_id=s.sid,
                     schedule_id=s.sched.schedule_id, denoise=s.denoise, hybrid=hybrid, decode_skipped=skipped,
                     rms_vs_reference=rms)
        self.completions += 1
        self.last = lat
        return rec

    def _refill(self):  # pipeline.py:495-521
        for i in range(self.depth):
            if self.slots[i] is not None:
                continue
            if not (self.warmup <= 0 or self.last_admit is None or self.tick_index - self.last_admit >= self.spacing):
                break
            if self.queue:
                sub = self.queue.popleft()
            elif self.auto and self.template is not None:
                self._enqueue(None)
                sub = self.queue.popleft()
            else:
                break
            self.slots[i] = self._admit(sub)
            if self.warmup > 0:
                self.warmup -= 1
            self.last_admit = self.tick_index

    def _admit(self, sub):  # pipeline.py:523-542
        sid, req, d, sched = sub
        stream = req.content_key()
        n = normal(self.seed, stream, 0, "init", (self.T, self.D))
        x = d * n + (1.0 - d) * req.source if d < 1.0 else n
        return Slot(sid, req, d, sched, x, self.steps, stream, self.tick_index)

    def render(self, req=None, denoise=None):  # pipeline.py:546-566
        req = req if req is not None else self.template
        d = self.denoise if denoise is None else denoise
        s = self._admit((-1, req, d, self.cache.get(d, self.steps, self.shift)))
        for _ in range(self.steps):
            self._step(s)
        return s.x.copy()


# --------------------------------------------------------------------- codec.py ---


def quantize(samples):  # codec.py:27-31
    scaled = samples * 32767
    r = np.copysign(np.floor(np.abs(scaled) + 0.5), scaled)
    return np.clip(r, -32768, 32767).astype(np.int16)


class Codec:
    """ToyCodec decoder (codec.py:67-164)."""

    def __init__(self, channels=8, hop=64, dilations=(1, 2, 4, 8), seed=7):
        self.C, self.hop, self.dil = channels, hop, tuple(dilations)
        self.rf = sum(self.dil)
        sc = 1.0 / np.sqrt(3 * channels)
        self.kernels = [normal(seed, 0, i, "decoder-conv", (3, channels, channels)) * sc for i in range(len(self.dil))]
        self.up = normal(seed, 0, 0, "decoder-up", (hop, channels)) * (0.5 / np.sqrt(channels))

    def _stack(self, h, valid=None):  # codec.py:93-125
        mask = None
        if valid is not None and (valid[0] > 0 or valid[1] < h.shape[0]):
            mask = np.zeros((h.shape[0], 1))
            mask[valid[0]:valid[1]] = 1.0
        for K, d in zip(self.kernels, self.dil):
            F = h.shape[0]
            p = np.zeros((F + 2 * d, h.shape[1]))
            p[d:d + F] = h
            h = np.tanh(p[0:F] @ K[0] + p[d:d + F] @ K[1] + p[2 * d:2 * d + F] @ K[2])
            if mask is not None:
                h = h * mask
        return h

    def full(self, latent):
        return quantize((self._stack(np.asarray(latent, dtype=np.float64)) @ self.up.T).reshape(-1))

    def window(self, latent, start, stop, ov):  # codec.py:136-164
        T = latent.shape[0]
        lo, hi = start - ov, stop + ov
        ext = np.zeros((hi - lo, latent.shape[1]))
        a, b = max(lo, 0), min(hi, T)
        ext[a - lo:b - lo] = latent[a:b]
        s = (self._stack(ext, (a - lo, b - lo)) @ self.up.T).reshape(-1)
        return quantize(s[ov * self.hop: ov * self.hop + (stop - start) * self.hop])
