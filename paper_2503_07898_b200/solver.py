"""Solver front-end: SolverConfig, run(config) -> RunResult on the B200 engines.

Mirrors proj/include/voxl/solver.hpp and proj/src/solver.cpp:
``config_from_json`` (:59-99) with ``SolverConfig::validate`` (:27-57),
``config_to_json`` (:101-119), ``run`` (:369-375) routing to the dense /
block-sparse / multires engines, and the result's artifact formats
(``diagnostics_csv`` :139-148, ledger CSV partition.cpp:89-96, trace JSON
:98-109, field header, dispatch JSON, graph DOT, distribution).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field as dc_field

import numpy as np

from ._capi import VoxlInstability

LATTICE_NAMES = ("D2Q9", "D3Q19", "D3Q27")
SCENARIOS = ("lid_driven_cavity", "flow_over_obstacle", "periodic_box")
LAYOUTS = ("AoS", "SoA", "DisagSoA")
STRATEGIES = ("naive", "disag_bitmask", "disag_mem")
Q_OF = {"D2Q9": 9, "D3Q19": 19, "D3Q27": 27}


class ConfigError(RuntimeError):
    """solver.hpp:23-25; the CLI maps it to exit code 2."""


@dataclass
class SolverConfig:
    lattice: str = "D3Q19"
    domain: tuple = (32, 32, 32)
    tau: float = 0.56
    scenario: str = "lid_driven_cavity"
    velocity: tuple = (0.05, 0.0, 0.0)
    steps: int = 200
    layout: str = "DisagSoA"
    partitions: int = 1
    strategy: str = "naive"
    obstacle_radius: float = 0.0
    levels: int = 1
    fused: bool = True
    seed: int = 42
    perturbation: float = 0.0
    # B200 execution options (not part of the reference schema)
    precision: str = "fp32"
    block_edge: int = 8

    def dim(self):
        return 2 if self.lattice == "D2Q9" else 3

    def partition_axis(self):
        return 1 if self.dim() == 2 else 2

    def validate(self):
        """SolverConfig::validate (solver.cpp:27-57), same messages."""
        err = []
        speed = math.sqrt(sum(v * v for v in self.velocity))
        nx, ny, nz = self.domain
        if not self.tau > 0.5:
            err.append("tau must be > 0.5; ")
        if speed > 0.1:
            err.append("|velocity| must be <= 0.1 (stability envelope); ")
        if self.steps < 0:
            err.append("steps must be >= 0; ")
        if nx < 2 or ny < 2:
            err.append("domain extents must be >= 2; ")
        if self.dim() == 2 and nz != 1:
            err.append("D2Q9 requires nz == 1; ")
        if self.dim() == 3 and nz < 2:
            err.append("3D lattices require nz >= 2; ")
        if self.partitions < 1:
            err.append("partitions must be >= 1; ")
        if self.partitions > 1 and self.domain[self.partition_axis()] < 2 * self.partitions:
            err.append("partition axis too small for the partition count; ")
        if self.levels < 1 or self.levels > 4:
            err.append("levels must be in [1, 4]; ")
        if self.levels > 1 and self.scenario != "lid_driven_cavity":
            err.append("multi-level runs support the lid_driven_cavity scenario only; ")
        if self.levels > 1 and self.partitions > 1:
            err.append("multi-level runs are single-partition; ")
        if self.levels > 1:
            scale = 1 << (self.levels - 1)
            if nx % scale or ny % scale or (self.dim() == 3 and nz % scale):
                err.append("domain extents must divide the coarsest cell size; ")
        if self.perturbation < 0.0 or self.perturbation > 0.5:
            err.append("perturbation must be in [0, 0.5]; ")
        if self.scenario == "flow_over_obstacle":
            mn = min(nx, ny, nz)
            r = self.obstacle_radius if self.obstacle_radius > 0.0 else mn / 5.0
            if 2.0 * r >= mn - 4:
                err.append("obstacle does not fit the domain; ")
        if err:
            raise ConfigError("invalid configuration: " + "".join(err))


def config_from_json(text: str) -> SolverConfig:
    """config_from_json (solver.cpp:59-99)."""
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise ConfigError(f"configuration is not valid JSON: {e}") from e
    c = SolverConfig()
    try:
        if "lattice" in j:
            if j["lattice"] not in LATTICE_NAMES:
                raise ConfigError("configuration error: unknown lattice kind: " + str(j["lattice"]))
            c.lattice = j["lattice"]
        if "domain" in j:
            d = j["domain"]
            if not isinstance(d, list) or len(d) < 2 or len(d) > 3:
                raise ConfigError("domain must be [nx, ny] or [nx, ny, nz]")
            c.domain = (int(d[0]), int(d[1]), int(d[2]) if len(d) == 3 else 1)
        if "tau" in j:
            c.tau = float(j["tau"])
        if "scenario" in j:
            if j["scenario"] not in SCENARIOS:
                raise ConfigError("unknown scenario: " + str(j["scenario"]))
            c.scenario = j["scenario"]
        if "velocity" in j:
            v = list(c.velocity)
            for a in range(min(3, len(j["velocity"]))):
                v[a] = float(j["velocity"][a])
            c.velocity = tuple(v)
        for key, cast in (("steps", int), ("partitions", int), ("obstacle_radius", float), ("levels", int),
                          ("seed", int), ("perturbation", float), ("block_edge", int)):
            if key in j:
                setattr(c, key, cast(j[key]))
        if "fused" in j:
            c.fused = bool(j["fused"])
        if "layout" in j:
            if j["layout"] not in LAYOUTS:
                raise ConfigError("configuration error: unknown layout scheme: " + str(j["layout"]))
            c.layout = j["layout"]
        if "strategy" in j:
            if j["strategy"] not in STRATEGIES:
                raise ConfigError("configuration error: unknown sparse strategy: " + str(j["strategy"]))
            c.strategy = j["strategy"]
        if "precision" in j:
            c.precision = str(j["precision"])
    except ConfigError:
        raise
    except Exception as e:  # noqa: BLE001 - mirror the reference's catch-all
        raise ConfigError(f"configuration error: {e}") from e
    c.validate()
    return c


def config_to_json(c: SolverConfig) -> str:
    """config_to_json (solver.cpp:101-119): nlohmann dump(2), keys sorted."""
    j = {"lattice": c.lattice,
         "domain": list(c.domain[:2]) if c.dim() == 2 else list(c.domain),
         "tau": c.tau, "scenario": c.scenario, "velocity": list(map(float, c.velocity)), "steps": c.steps,
         "layout": c.layout, "partitions": c.partitions, "strategy": c.strategy, "levels": c.levels,
         "fused": c.fused, "seed": c.seed, "perturbation": c.perturbation}
    if c.obstacle_radius > 0.0:
        j["obstacle_radius"] = c.obstacle_radius
    text = json.dumps(j, indent=2, sort_keys=True)
    # nlohmann 3.11.3 prints the domain array (built with json::array({...}))
    # on one line without spaces; reproduce that byte for byte.
    import re

    text = re.sub(r'"domain": \[\s*([^\]]*?)\s*\]',
                  lambda m: '"domain": [' + ",".join(x.strip() for x in m.group(1).split(",")) + "]", text)
    return text + "\n"


@dataclass
class RunResult:
    config: SolverConfig
    field: np.ndarray = None
    field_header_json: str = ""
    diagnostics: list = dc_field(default_factory=list)  # (step, mass, max_speed)
    ledger: list = dc_field(default_factory=list)       # TransferRecord
    trace: list = dc_field(default_factory=list)        # (step, stage, phase, partition)
    dispatch_json: str = ""
    graph_dot: str = ""
    distribution: str = ""
    observed_trace_json: str = ""  # the executed schedule (run(..., observed_trace=True), dense path)

    def diagnostics_csv(self) -> str:
        """solver.cpp:139-148 (%.17g)."""
        rows = ["step,mass,max_u\n"]
        rows += ["%d,%.17g,%.17g\n" % (s, m, u) for s, m, u in self.diagnostics]
        return "".join(rows)

    def ledger_csv(self) -> str:
        """TransferLedger::to_csv (partition.cpp:89-96)."""
        out = ["step,src,dst,base_src,base_dst,elements\n"]
        out += [f"{r.step},{r.src},{r.dst},{r.base_src},{r.base_dst},{r.elements}\n" for r in self.ledger]
        return "".join(out)

    def trace_json(self) -> str:
        """TraceLog::to_json (partition.cpp:98-109)."""
        lines = ["[\n"]
        for i, (step, stage, phase, p) in enumerate(self.trace):
            sep = "," if i + 1 < len(self.trace) else ""
            lines.append(f'  {{"step": {step}, "stage": {stage}, "phase": "{phase}", "partition": {p}}}{sep}\n')
        lines.append("]\n")
        return "".join(lines)


BAD_DENSITY = 31  # voxl_diag.bad_population of a non-positive density (VOXL_BAD_DENSITY)


def _unstable(d, step):
    """run()'s abort for one probe row (the per-step loop shape)."""
    if not d.unstable:
        return
    if d.bad_population == BAD_DENSITY:  # macroscopic's throw inside probe_field (lattice.cpp:124)
        raise RuntimeError(f"run aborted at step {step}: macroscopic: non-positive density")
    raise RuntimeError(f"run aborted at step {step}: instability at step {step}, voxel {d.bad_voxel}, "
                       f"population {d.bad_population}")


def _probed_rows(eng, steps):
    """n probed steps through the engine's fused step_probe_n: (rows, error)
    -- the rows of the steps that completed and run()'s abort text, if any."""
    try:
        return eng.step_probe_n(steps), None
    except VoxlInstability as e:
        return e.rows, e


def run_dense(c: SolverConfig, observed_trace: bool = False) -> RunResult:
    """run_dense (solver.cpp:225-266) on DenseEngine. observed_trace: also
    record the executed step schedule (voxl_dense_trace_json: every launched
    phase with its stream, device and CUDA-event times)."""
    from .dense import DenseEngine, plan_ledger
    from .initial import initial_canonical_state

    r = RunResult(config=c)
    eng = DenseEngine(lattice=c.lattice, domain=c.domain, tau=c.tau, scenario=c.scenario, velocity=c.velocity,
                      layout=c.layout, partitions=c.partitions, precision=c.precision)
    eng.set_canonical(initial_canonical_state(c))
    if observed_trace:
        eng.trace(True)
    # step_occ + probe_field per step, fused on the device; rows read back per
    # batch, the first failing step raises run()'s text
    rows, err = _probed_rows(eng, c.steps)
    if observed_trace:
        r.observed_trace_json = eng.trace_json()
        eng.trace(False)
    for step, d in enumerate(rows):
        r.diagnostics.append((step, d.mass, d.max_speed))
        r.ledger += plan_ledger(step, lattice=c.lattice, domain=c.domain, layout=c.layout, partitions=c.partitions,
                                scenario=c.scenario)
        r.trace += [(step, 1, "halo", p) for p in range(c.partitions)]
        r.trace += [(step, 1, "private", p) for p in range(c.partitions)]
        r.trace += [(step, 2, "shared", p) for p in range(c.partitions)]
    if err is not None:
        eng.close()
        raise RuntimeError(str(err))
    r.field = eng.get_canonical()
    eng.close()
    nx, ny, nz = c.domain
    r.field_header_json = (f'{{"shape": [{nx}, {ny}, {nz}], "lattice": "{c.lattice}", "representation": "dense", '
                           f'"layout": "{c.layout}", "cardinality": {Q_OF[c.lattice]}, '
                           f'"order": "voxel-major (x fastest), component innermost"}}\n')
    return r


def run_sparse(c: SolverConfig) -> RunResult:
    """run_sparse (solver.cpp:268-310) on SparseEngine."""
    from .sparse import SparseEngine, obstacle_mask

    r = RunResult(config=c)
    act = obstacle_mask(c.domain, c.obstacle_radius)
    eng = SparseEngine(c.domain, act, tau=c.tau, u_bc=c.velocity, block_edge=c.block_edge, strategy=c.strategy,
                       precision=c.precision, lattice=c.lattice)
    rows, err = _probed_rows(eng, c.steps)  # step + probe_field, fused on the device
    r.diagnostics = [(step, d.mass, d.max_speed) for step, d in enumerate(rows)]
    if err is not None:
        eng.close()
        raise RuntimeError(str(err))
    r.field = eng.get_state()
    # The report is the reference's (edge-4 tables); the engine's own blocks may be 8^3.
    from .sparse import SparsePlan

    r.dispatch_json = SparsePlan(c.domain, act, block_edge=4, strategy=c.strategy, lattice=c.lattice).report_json() \
        + "\n"
    nx, ny, nz = c.domain
    r.field_header_json = (f'{{"shape": [{nx}, {ny}, {nz}], "lattice": "{c.lattice}", '
                           f'"representation": "block_sparse", "strategy": "{c.strategy}", '
                           f'"cardinality": {Q_OF[c.lattice]}, "active_voxels": {int(act.sum())}, '
                           f'"order": "active cells sorted by (z, y, x), component innermost"}}\n')
    eng.close()
    return r


def run_multires(c: SolverConfig) -> RunResult:
    """run_multires (solver.cpp:312-367) on MultiResEngine."""
    from .multires import MultiResEngine, MultiResPlan, band_level_map

    r = RunResult(config=c)
    lm = band_level_map(c.domain, c.levels, c.partition_axis())
    eng = MultiResEngine(c.domain, c.levels, level_map=lm, tau=c.tau, lid_u=c.velocity, fused=c.fused,
                         precision=c.precision, block_edge=c.block_edge, lattice=c.lattice)
    # coarse_step + probe_field, the probe fused into each level's last sub-step
    rows, err = _probed_rows(eng, c.steps)
    r.diagnostics = [(step, d.mass, d.max_speed) for step, d in enumerate(rows)]
    if err is not None:
        eng.close()
        raise RuntimeError(str(err))
    r.field = eng.get_state()
    plan = MultiResPlan(c.domain, c.levels, level_map=lm, tau=c.tau, lattice=c.lattice)
    r.graph_dot = plan.graph_dot(fused=c.fused)
    r.distribution = plan.distribution() + "\n"
    nx, ny, nz = c.domain
    r.field_header_json = (f'{{"shape": [{nx}, {ny}, {nz}], "lattice": "{c.lattice}", '
                           f'"representation": "multires", "levels": {c.levels}, "cardinality": {Q_OF[c.lattice]}, '
                           f'"order": "levels finest to coarsest, cells sorted by (z, y, x), component innermost"}}\n')
    eng.close()
    return r


def run(c: SolverConfig, observed_trace: bool = False) -> RunResult:
    """run (solver.cpp:369-375). observed_trace: the dense route also records
    the executed step schedule (RunResult.observed_trace_json)."""
    c.validate()
    if c.levels > 1:
        return run_multires(c)
    if c.scenario == "flow_over_obstacle":
        return run_sparse(c)
    return run_dense(c, observed_trace)


def write_outputs(result: RunResult, out_dir: str) -> None:
    """cmd_run's artifact set (tools/main.cpp:30-55)."""
    import os

    os.makedirs(out_dir, exist_ok=True)
    result.field.astype(np.float64).tofile(os.path.join(out_dir, "fields.bin"))

    def w(name, text):
        with open(os.path.join(out_dir, name), "w") as f:
            f.write(text)

    w("fields.json", result.field_header_json)
    w("diagnostics.csv", result.diagnostics_csv())
    w("config.json", config_to_json(result.config))
    if result.ledger:
        w("ledger.csv", result.ledger_csv())
    if result.trace:
        w("trace.json", result.trace_json())
    if result.observed_trace_json:
        w("trace_observed.json", result.observed_trace_json)
    if result.dispatch_json:
        w("dispatch.json", result.dispatch_json)
    if result.graph_dot:
        w("graph.dot", result.graph_dot)
    if result.distribution:
        w("distribution.txt", result.distribution)
