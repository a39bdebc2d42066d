"""pytest plugin: run the reference's OWN test suites through the B200 path.

SURVEY §8(c) "running the reference's own tests against the drop-in": loaded
with ``-p tools.refpatch`` before the reference's test modules are collected,
it rebinds the hot-path entry points -- in their defining modules, in the
package re-exports (``gpukalc/__init__.py:65-71``) and in the CLI modules that
imported them by name -- to thin adapters over this package's device API, so
the unmodified reference tests call the CUDA kernels:

* ``gpukalc.scheduler.schedule_block`` / ``schedule_cfg`` / ``schedule_kernel``
  (``scheduler.py:137-363``) -> K1 + fused K2/K3 (``schedule_batch``, trace on);
* ``gpukalc.features.extract_features`` (``features.py:149-247``) -> same launch;
* ``gpukalc.features.features_to_csv`` / ``features_from_csv``
  (``features.py:250-272``) -> the native CSV writer / parser (``gk_featio``);
* ``gpukalc.power.load_ensemble`` (``power.py:73-125``) -> native loader
  (``gk_ensio``), ``predict_power`` (``power.py:148-168``) -> K4;
* ``gpukalc_trainer.training._make_model`` (``training.py:65-79``) -> the K5
  estimators (``forest.RandomForestRegressor``, ``boosting.GradientBoostingRegressor``);
* ``gpukalc_trainer.dataset.prune_correlated`` (``dataset.py:138-183``) ->
  ``pruning.prune_correlated`` (GPU correlation matrix).

The adapters only convert types: results come back as the reference's own
frozen dataclasses and errors as the reference's exception classes with this
package's (reference-identical) messages.  Nothing falls back to the
reference's implementation -- a device failure fails the test.

Test infrastructure, like ``oracle/``: run by ``tools/refsuite.sh`` (GPU box),
never imported by the product.
"""

from __future__ import annotations

import functools

import gpukalc
import gpukalc.cli as ref_cli
import gpukalc.errors as ref_errors
import gpukalc.features as ref_features
import gpukalc.power as ref_power
import gpukalc.scheduler as ref_sched
from gpukalc.ptx.types import InstClass, KernelGraph

import paper_2305_01886_b200 as gk
from paper_2305_01886_b200 import abi
from paper_2305_01886_b200 import errors as gk_errors

PATCHED: list = []


def _translate(fn):
    """Re-raise this package's exceptions as the reference's same-named ones."""

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        try:
            return fn(*args, **kwargs)
        except gk_errors.DeviceError:
            raise
        except gk_errors.TrainerError as exc:
            from gpukalc_trainer.errors import TrainerError

            raise TrainerError(str(exc)) from exc
        except gk_errors.GpukalcError as exc:
            raise getattr(ref_errors, type(exc).__name__)(str(exc)) from exc

    return wrapper


# ------------------------------------------------------------- scheduler


def _trace(profile, graph, launch, n_tw=None, gm=None):
    """One point through the device with per-instruction trace rows."""
    from paper_2305_01886_b200 import api, runtime

    if n_tw is None:
        return api.schedule_batch([profile], [graph], [launch], features=False, trace=True)
    dc = api._device_corpus([graph])
    dg = runtime.DeviceGrid.build(dc, [profile], [(1, 32, 0, 0)], n_tw=[n_tw], gm=[gm])
    out = runtime.schedule_features(dc, dg, trace=True)
    return {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in out.items()}


def _blocks(graph, out) -> tuple:
    blocks, t = [], 0
    for b, blk in enumerate(graph.blocks):
        rows = []
        for i, ins in enumerate(blk.instructions):
            rows.append(ref_sched.InstSchedule(
                index=i, opcode=ins.opcode, klass=ins.klass, resource=ins.resource,
                start=float(out["tr_start"][0, t]), duration=float(out["tr_duration"][0, t]),
                latency=float(out["tr_latency"][0, t]), n_batches=int(out["tr_n_batches"][0, t])))
            t += 1
        blocks.append(ref_sched.BlockSchedule(label=blk.label, rows=tuple(rows),
                                              delay=float(out["tr_blk_delay"][0, b])))
    return tuple(blocks)


def _gm_for(profile, graph, gm_latency):
    """``latency_of``'s GLOBAL rule (profiles.py:196-204) for the n_tw faces."""
    if gm_latency is not None:
        return float(gm_latency)
    table = profile.latency.instructions
    if "global" in table:
        return float(table["global"])
    if any(i.klass is InstClass.GLOBAL for b in graph.blocks for i in b.instructions):
        raise ref_errors.ProfileError(
            "global-memory latency unresolved: pass gm_latency or add a 'global' latency entry")
    return 0.0


@_translate
def schedule_block(profile, block, n_tw, *, gm_latency=None):
    if n_tw < 1:
        raise ref_errors.ScheduleError("thread count must be >= 1")
    graph = KernelGraph(name="block", blocks=[block])
    out = _trace(profile, graph, None, n_tw, _gm_for(profile, graph, gm_latency))
    return _blocks(graph, out)[0]


@_translate
def schedule_cfg(profile, graph, n_tw, *, gm_latency=None):
    if n_tw < 1:
        raise ref_errors.ScheduleError("thread count must be >= 1")
    mult = graph.loop_multipliers()
    graph.topo_order()          # the reference's cyclic-CFG error, same point
    out = _trace(profile, graph, None, n_tw, _gm_for(profile, graph, gm_latency))
    return ref_sched.CfgSchedule(
        blocks=_blocks(graph, out), multipliers=tuple(mult),
        finish=tuple(float(v) for v in out["tr_blk_finish"][0]),
        delay=float(out["sf"][0][abi.SF_NAMES.index("cfg_delay")]))


@_translate
def schedule_kernel(profile, graph, launch):
    ks = gk.schedule_kernel(profile, graph, launch)
    c = ks.cfg
    cfg = ref_sched.CfgSchedule(blocks=_blocks_from(graph, c), multipliers=c.multipliers,
                                finish=c.finish, delay=c.delay)
    return ref_sched.KernelSchedule(
        kernel=ks.kernel, launch=launch, threads_scheduled=ks.threads_scheduled,
        threads_per_sm=ks.threads_per_sm, blocks_per_sm=ks.blocks_per_sm, waves=ks.waves,
        gm_latency=ks.gm_latency, cfg=cfg, d_kernel=ks.d_kernel,
        overhead_cycles=ks.overhead_cycles, gm_penalty=ks.gm_penalty, sm_penalty=ks.sm_penalty,
        cm_penalty=ks.cm_penalty, n_global=ks.n_global, n_shared=ks.n_shared)


def _blocks_from(graph, cfg) -> tuple:
    out = []
    for blk, bs in zip(graph.blocks, cfg.blocks):
        rows = tuple(ref_sched.InstSchedule(
            index=r.index, opcode=r.opcode, klass=ins.klass, resource=ins.resource,
            start=r.start, duration=r.duration, latency=r.latency, n_batches=r.n_batches)
            for r, ins in zip(bs.rows, blk.instructions))
        out.append(ref_sched.BlockSchedule(label=bs.label, rows=rows, delay=bs.delay))
    return tuple(out)


@_translate
def extract_features(profile, graph, launch):
    fv = gk.extract_features(profile, graph, launch)
    return ref_features.FeatureVector(*fv.as_row())


def features_to_csv(rows, *, selected=False):
    return gk.features_to_csv(rows, selected=selected)


def features_from_csv(text):
    return gk.features_from_csv(text)


# ----------------------------------------------------------------- power

_ENS: dict = {}


def _ours(ens):
    """Reference TreeEnsemble -> this package's (same fields), cached by identity."""
    if isinstance(ens, gk.TreeEnsemble):
        return ens
    hit = _ENS.get(id(ens))
    if hit is None or hit[0] is not ens:
        hit = _ENS[id(ens)] = (ens, gk.TreeEnsemble(
            base_score=ens.base_score, feature_manifest=tuple(ens.feature_manifest),
            scale_min=tuple(ens.scale_min), scale_max=tuple(ens.scale_max),
            trees=ens.trees, gains=tuple(ens.gains)))
    return hit[1]


@_translate
def load_ensemble(source):
    e = gk.load_ensemble(source)
    ref = ref_power.TreeEnsemble(
        base_score=e.base_score, feature_manifest=tuple(e.feature_manifest),
        scale_min=tuple(e.scale_min), scale_max=tuple(e.scale_max),
        trees=tuple(tuple(t) for t in e.trees), gains=tuple(e.gains))
    _ENS[id(ref)] = (ref, e)    # keep the native loader's device layout
    return ref


@_translate
def predict_power(ensemble, features):
    return gk.predict_power(_ours(ensemble), features)


# --------------------------------------------------------------- trainer


def _make_model(family, n_estimators, learning_rate, max_depth, seed):
    from paper_2305_01886_b200.boosting import GradientBoostingRegressor
    from paper_2305_01886_b200.forest import RandomForestRegressor

    if family == "gradient_boosted":
        kwargs = {} if max_depth is None else {"max_depth": max_depth}
        return GradientBoostingRegressor(n_estimators=n_estimators, learning_rate=learning_rate,
                                         random_state=seed, **kwargs)
    if family == "random_forest":
        return RandomForestRegressor(n_estimators=n_estimators, max_depth=max_depth,
                                     random_state=seed)
    from gpukalc_trainer.errors import TrainerError

    raise TrainerError(f"unknown model family '{family}'")


@_translate
def prune_correlated(dataset, method="pearson", threshold=0.85):
    from gpukalc_trainer import dataset as ref_ds

    from paper_2305_01886_b200 import pruning

    out, drops = pruning.prune_correlated(dataset, method, threshold)
    return out, [ref_ds.DropEntry(d.dropped, d.kept, d.method, d.coefficient) for d in drops]


# ----------------------------------------------------------------- patch


def _rebind(modules, name, fn):
    for m in modules:
        if hasattr(m, name):
            setattr(m, name, fn)
            PATCHED.append(f"{m.__name__}.{name}")


def _warm() -> None:
    """Create the CUDA context and load the kernels once, at plugin load (what a
    long-lived caller pays at start-up), so the suites' wall-clock asserts
    (e.g. test_acceptance.py:65) time the calls, not driver initialisation."""
    from gpukalc.profiles import profile_from_dict  # noqa: F401
    from gpukalc.ptx import parse_ptx

    g = parse_ptx(".entry w() {\n\tld.global.f32 %f1, [%rd1];\n\tadd.f32 %f2, %f1, %f1;\n"
                  "\tst.shared.f32 [%rd2], %f2;\n\tret;\n}\n", "w")
    gk.extract_features(gk.resolve_profile("tesla_k20"), g, gk.LaunchConfig(13, 128, 32, 0))


def install(trainer: bool = True, warm: bool = True) -> None:
    import paper_2305_01886_b200.runtime as rt

    rt.load_library()           # the CUDA library must be there: no silent host path
    if warm:
        _warm()
    inf = [gpukalc, ref_sched, ref_features, ref_power, ref_cli]
    _rebind(inf, "schedule_block", schedule_block)
    _rebind(inf, "schedule_cfg", schedule_cfg)
    _rebind(inf, "schedule_kernel", schedule_kernel)
    _rebind(inf, "extract_features", extract_features)
    _rebind(inf, "features_to_csv", features_to_csv)
    _rebind(inf, "features_from_csv", features_from_csv)
    _rebind(inf, "load_ensemble", load_ensemble)
    _rebind(inf, "predict_power", predict_power)
    if trainer:
        try:
            import gpukalc_trainer
            import gpukalc_trainer.cli as tcli
            import gpukalc_trainer.dataset as tds
            import gpukalc_trainer.training as ttr
        except ImportError:
            return
        _rebind([ttr], "_make_model", _make_model)
        _rebind([gpukalc_trainer, tds, tcli], "prune_correlated", prune_correlated)


def pytest_configure(config):
    install()


def pytest_terminal_summary(terminalreporter):
    from paper_2305_01886_b200.runtime import LIB_PATH

    terminalreporter.write_line(f"refpatch: {LIB_PATH} bound for " + ", ".join(PATCHED))
