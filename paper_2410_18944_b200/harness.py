"""The callers of the path: the reference's harness
(proj/src/solver.cpp:92-332, proj/include/wost/solver.hpp) re-linked to the
GPU path, plus its result formats (proj/src/image.cpp:46-230).

  run_solve(cfg)                 -> RunResult        solver.cpp:124-167
  solve_points(prob, cfg, xy, w) -> ProbeResult      solver.cpp:108-122
  generate_reference(cfg, wpp)   -> SolutionImage    solver.cpp:169-190
  run_ablation(cfg, modes, ref)  -> [AblationRow]    solver.cpp:192-232
  run_equal_time(cfg, modes, ref, seconds)           new: the paper's equal-time
                                                      comparison (SPEC.md cfg 2)
  parse_run_config / load_run_config_file            solver.cpp:244-315
  write_csv / read_csv / write_pfm / read_pfm /
  write_png / compute_relmse / write_convergence_log image.cpp, solver.cpp:317-327

The Engine loop is the reference's: round b runs one walk per point with walk
streams (seed, point, b), and trains on the round's records while
b < train_until (training_active, guide_train.cpp:200-202). Each round is
enqueued on the device (wostgpu_solve_rounds + wostgpu_train_round); the host
only reads the statistics back to log relMSE, exactly when the reference
computes it. Times are wall-clock seconds like the reference's log.
"""
from __future__ import annotations

import dataclasses
import json
import math
import struct
import time
import zlib
from typing import Callable, List, Optional

import numpy as np

from . import abi, api
from .scene import Scene, cell_centers, make_preset

def parse_sampler_mode(s: str) -> str:
    """parse_sampler_mode (wost.cpp): the names the reference accepts."""
    if s not in abi.MODES:
        raise ValueError(f"unknown sampler mode '{s}'")
    return s


# ---------------------------------------------------------------- config
@dataclasses.dataclass
class RunConfig:
    """wost::RunConfig (solver.hpp:18-42)."""
    scene_path: str = ""
    preset: str = ""
    width: int = 128
    height: int = 128
    bbox: Optional[tuple] = None  # empty: preset eval bbox, then scene bbox
    wpp: int = 256
    mode: str = "uniform"
    fixed_c: float = 0.5
    train_until: int = 256
    field: abi.FieldConfig = dataclasses.field(default_factory=abi.field_config)
    train: abi.TrainConfig = dataclasses.field(default_factory=abi.train_config)
    rr_depth: int = 128
    reflect: bool = True
    epsilon_shell: float = 0.0
    r_min: float = 0.0
    clamp_grazing: bool = False
    seed: int = 1
    out_csv: str = ""
    out_pfm: str = ""
    out_png: str = ""
    log_path: str = ""
    reference_path: str = ""
    field_in: str = ""
    field_out: str = ""
    mlp: int = api.MLP_TENSOR  # device MLP path of the guided walks

    def solver_config(self) -> abi.SolverConfig:
        return abi.solver_config(self.mode, epsilon_shell=self.epsilon_shell, r_min=self.r_min,
                                 rr_depth=self.rr_depth, fixed_c=self.fixed_c, reflect=self.reflect,
                                 clamp_grazing=self.clamp_grazing)


def parse_run_config(text: str) -> RunConfig:
    """parse_run_config (solver.cpp:244-305): same keys, defaults and checks."""
    doc = json.loads(text)
    cfg = RunConfig()
    cfg.scene_path = doc.get("scene", "")
    cfg.preset = doc.get("preset", "")
    g = doc.get("grid", {})
    cfg.width = int(g.get("width", cfg.width))
    cfg.height = int(g.get("height", cfg.height))
    if isinstance(g.get("bbox"), dict):
        b = g["bbox"]
        cfg.bbox = (float(b["min"][0]), float(b["min"][1]), float(b["max"][0]), float(b["max"][1]))
    cfg.wpp = int(doc.get("wpp", cfg.wpp))
    if cfg.wpp < 1:
        raise ValueError("run config: wpp must be >= 1")
    if cfg.width < 1 or cfg.height < 1:
        raise ValueError("run config: grid resolution must be >= 1x1")
    if "sampler" in doc:
        cfg.mode = parse_sampler_mode(doc["sampler"])
    cfg.fixed_c = float(doc.get("fixed_c", cfg.fixed_c))
    if not 0.0 < cfg.fixed_c < 1.0:
        raise ValueError("run config: fixed_c must lie in (0,1)")
    cfg.train_until = int(doc.get("train_until", cfg.train_until))
    cfg.seed = int(doc.get("seed", cfg.seed))
    k = int(doc.get("k", cfg.field.mixture_k))
    f = doc.get("field", {})
    levels = tuple(f.get("levels", [cfg.field.level_res[i] for i in range(cfg.field.n_levels)]))
    cfg.field = abi.field_config(levels, features=int(f.get("features", cfg.field.features)),
                                 hidden=int(f.get("hidden", cfg.field.hidden)), mixture_k=k)
    t = doc.get("train", {})
    cfg.train = abi.train_config(minibatch=int(t.get("minibatch", cfg.train.minibatch)),
                                 max_records=int(t.get("max_records", cfg.train.max_records_per_round)),
                                 lr=float(t.get("lr", cfg.train.lr)),
                                 e_fraction=float(t.get("e_fraction", cfg.train.e_fraction)))
    s = doc.get("solver", {})
    cfg.rr_depth = int(s.get("rr_depth", cfg.rr_depth))
    cfg.reflect = bool(s.get("reflect", cfg.reflect))
    cfg.epsilon_shell = float(s.get("epsilon_shell", cfg.epsilon_shell))
    cfg.r_min = float(s.get("r_min", cfg.r_min))
    cfg.clamp_grazing = bool(s.get("clamp_grazing", cfg.clamp_grazing))
    cfg.out_csv = doc.get("out", "")
    cfg.out_pfm = doc.get("out_pfm", "")
    cfg.out_png = doc.get("out_png", "")
    cfg.log_path = doc.get("log", "")
    cfg.reference_path = doc.get("reference", "")
    cfg.field_in = doc.get("field_in", "")
    cfg.field_out = doc.get("field_out", "")
    return cfg


def load_run_config_file(path: str) -> RunConfig:
    with open(path, "rb") as f:
        return parse_run_config(f.read().decode())


# ---------------------------------------------------------------- problem
@dataclasses.dataclass
class Problem:
    """wost::Problem (solver.hpp:44-50)."""
    scene: Scene
    analytic: Optional[Callable[[float, float], float]]
    eval_bbox: tuple


def load_problem(cfg: RunConfig) -> Problem:
    """load_problem (solver.cpp): a preset, or a scene JSON file (scene_io.py)."""
    if not cfg.scene_path and not cfg.preset:
        raise ValueError("run config needs a 'preset' or a 'scene'")
    if cfg.preset:  # the preset wins when both are set (solver.cpp:30-41)
        p = make_preset(cfg.preset)
        return Problem(p.scene, p.analytic, p.eval_bbox)
    from .scene_io import load_scene_file
    sc = load_scene_file(cfg.scene_path)
    return Problem(sc, None, sc.bbox)


def grid_bbox(cfg: RunConfig, prob: Problem) -> tuple:
    return tuple(cfg.bbox) if cfg.bbox is not None else tuple(prob.eval_bbox)


# ---------------------------------------------------------------- images
@dataclasses.dataclass
class SolutionImage:
    """wost::SolutionImage (image.hpp): PointStats per cell, row-major j*w+i."""
    width: int
    height: int
    bbox: tuple
    cells: np.ndarray  # abi.POINT_STATS_DTYPE

    def cell_centers(self):
        return cell_centers(self.width, self.height, self.bbox)

    @property
    def mean(self):
        return self.cells["mean"]

    def variance_of_mean(self):
        c = self.cells["count"].astype(np.float64)
        return np.where(c > 1, self.cells["m2"] / np.maximum(c * (c - 1), 1.0), 0.0)


def make_image(width, height, bbox) -> SolutionImage:
    return SolutionImage(width, height, tuple(bbox), np.zeros(width * height, dtype=abi.POINT_STATS_DTYPE))


def compute_relmse(est: SolutionImage, ref: SolutionImage) -> float:
    """compute_relmse (image.cpp:211-230), including the +inf case."""
    if est.width != ref.width or est.height != ref.height:
        raise ValueError("compute_relmse: image dimensions differ")
    r = ref.mean
    max_abs = float(np.max(np.abs(r))) if r.size else 0.0
    delta = 0.0001 * max_abs * max_abs
    d = est.mean - r
    denom = r * r + delta
    bad = denom <= 0.0
    if np.any(bad & (d != 0.0)):
        return math.inf
    terms = np.where(bad, 0.0, d * d / np.where(bad, 1.0, denom))
    total = float(np.cumsum(terms)[-1]) if terms.size else 0.0  # sequential, like the reference loop
    return total / est.mean.size


def _g17(v: float) -> str:
    return "%.17g" % v


def write_csv(img: SolutionImage, path: str):
    """write_csv (image.cpp:46-62): '%.17g' values, i,j,mean,var,count."""
    var = img.variance_of_mean()
    lines = [f"# width={img.width} height={img.height} bbox=" + ",".join(_g17(v) for v in img.bbox),
             "i,j,mean,var,count"]
    for j in range(img.height):
        for i in range(img.width):
            k = j * img.width + i
            lines.append(f"{i},{j},{_g17(img.cells['mean'][k])},{_g17(var[k])},{int(img.cells['count'][k])}")
    with open(path, "w", newline="\n") as f:
        f.write("\n".join(lines) + "\n")


def read_csv(path: str) -> SolutionImage:
    """read_csv (image.cpp:64-92): m2 reconstructed so var round-trips."""
    with open(path) as f:
        header = f.readline()
        if not header.startswith("# width="):
            raise ValueError(f"{path}: bad csv header")
        parts = dict(kv.split("=") for kv in header[2:].split())
        w, h = int(parts["width"]), int(parts["height"])
        bbox = tuple(float(x) for x in parts["bbox"].split(","))
        img = make_image(w, h, bbox)
        f.readline()
        for line in f:
            i, j, mean, var, count = line.strip().split(",")
            k = int(j) * w + int(i)
            c = int(count)
            img.cells["mean"][k] = float(mean)
            img.cells["count"][k] = c
            img.cells["m2"][k] = float(var) * c * (c - 1) if c > 1 else 0.0
    return img


def write_pfm(img: SolutionImage, path: str):
    """write_pfm (image.cpp:94-107): 'Pf', little-endian fp32, row 0 first."""
    with open(path, "wb") as f:
        f.write(f"Pf\n{img.width} {img.height}\n-1.0\n".encode())
        f.write(img.mean.astype("<f4").tobytes())


def read_pfm(path: str) -> SolutionImage:
    with open(path, "rb") as f:
        data = f.read()
    toks = data.split(maxsplit=4)
    if toks[0] != b"Pf":
        raise ValueError(f"{path}: not a grayscale PFM")
    w, h, scale = int(toks[1]), int(toks[2]), float(toks[3])
    if scale >= 0.0:
        raise ValueError(f"{path}: big-endian PFM is not supported")
    raster = data[len(data) - 4 * w * h:]
    img = make_image(w, h, (0.0, 0.0, 1.0, 1.0))
    img.cells["mean"] = np.frombuffer(raster, "<f4").astype(np.float64)
    img.cells["count"] = 1
    return img


def write_png(img: SolutionImage, path: str, range_min=0.0, range_max=0.0):
    """write_png (image.cpp:155-209): 8-bit gray, top row first, deflate level
    9, plus the '<path>.json' tonemap sidecar."""
    m = img.mean
    if range_min == range_max:
        range_min, range_max = float(np.min(m)), float(np.max(m))
        if range_min >= range_max:
            range_max = range_min + 1.0
    t = np.clip((m.reshape(img.height, img.width) - range_min) / (range_max - range_min), 0.0, 1.0)
    px = np.floor(t * 255.0 + 0.5).astype(np.uint8)[::-1]  # std::lround, top row first
    raster = b"".join(b"\0" + row.tobytes() for row in px)

    def chunk(tag, payload):
        body = tag + payload
        return struct.pack(">I", len(payload)) + body + struct.pack(">I", zlib.crc32(body) & 0xFFFFFFFF)

    with open(path, "wb") as f:
        f.write(b"\x89PNG\r\n\x1a\n")
        f.write(chunk(b"IHDR", struct.pack(">IIBBBBB", img.width, img.height, 8, 0, 0, 0, 0)))
        f.write(chunk(b"IDAT", zlib.compress(raster, 9)))
        f.write(chunk(b"IEND", b""))
    with open(path + ".json", "w") as f:
        f.write(json.dumps({"tonemap": {"max": range_max, "min": range_min}}, indent=2) + "\n")


@dataclasses.dataclass
class LogRow:
    wpp: int
    relmse: float
    seconds: float


def write_convergence_log(rows: List[LogRow], path: str):
    """write_convergence_log (solver.cpp:317-327): 'wpp,relmse,seconds'."""
    with open(path, "w", newline="\n") as f:
        f.write("wpp,relmse,seconds\n")
        for r in rows:
            f.write("%d,%.9g,%.3f\n" % (r.wpp, r.relmse, r.seconds))


# ---------------------------------------------------------------- engine
class Engine:
    """Engine (solver.cpp:53-105) on the device: scene + BVH + field + solver."""

    def __init__(self, prob: Problem, cfg: RunConfig, points):
        self.cfg = cfg
        self.accel = api.Accel(prob.scene)
        self.guided = cfg.mode != "uniform"
        self.field = None
        if self.guided:
            if cfg.field_in:
                self.field = api.GuidingField.load(cfg.field_in)
            else:  # field seed = run seed (solver.cpp:80)
                self.field = api.GuidingField(cfg.field, prob.scene.bbox, cfg.seed)
        self.solver = api.Solver(self.accel, self.field, cfg.solver_config(), cfg.mlp)
        self.solver.set_points(points)
        self.train_totals = abi.TrainStats()
        # tcfg (solver.cpp:84-87): reflection follows the solver, the
        # selection loss trains only under learnable MIS, seed = run seed
        self.tcfg = abi.TrainConfig.from_buffer_copy(cfg.train)
        self.tcfg.reflect = int(cfg.reflect)
        self.tcfg.learn_selection = int(cfg.mode == "learnable_mis")
        self.tcfg.seed = cfg.seed

    def run_batch(self, rnd: int):
        """Engine::run_batch (solver.cpp:92-104): one walk per point, then
        train on the round's records while training is active."""
        training = self.guided and rnd < self.cfg.train_until
        self.solver.solve_rounds(self.cfg.seed, rnd, 1, collect=training)
        if training:
            st = self.solver.train_round(self.tcfg, rnd)
            for k in ("records_seen", "records_consumed", "skipped_low_pdf", "skipped_low_v", "steps"):
                setattr(self.train_totals, k, getattr(self.train_totals, k) + getattr(st, k))
            self.train_totals.seconds += st.seconds

    def stats(self):
        return self.solver.stats()


@dataclasses.dataclass
class RunResult:
    """wost::RunResult (solver.hpp:58-66)."""
    image: SolutionImage
    log: List[LogRow]
    seconds: float
    train_stats: abi.TrainStats
    escaped_walks: int
    field: Optional[api.GuidingField]


def run_solve(cfg: RunConfig) -> RunResult:
    """run_solve (solver.cpp:124-167): the full grid solve, relMSE logged
    after every round against the reference image when one is given."""
    t0 = time.perf_counter()
    prob = load_problem(cfg)
    img = make_image(cfg.width, cfg.height, grid_bbox(cfg, prob))
    eng = Engine(prob, cfg, img.cell_centers())
    reference = read_csv(cfg.reference_path) if cfg.reference_path else None
    log = []
    for b in range(cfg.wpp):
        eng.run_batch(b)
        rel = math.nan
        if reference is not None:
            img.cells = eng.stats()
            rel = compute_relmse(img, reference)
        log.append(LogRow(b + 1, rel, time.perf_counter() - t0))
    img.cells = eng.stats()
    out = RunResult(img, log, time.perf_counter() - t0, eng.train_totals,
                    int(img.cells["escaped"].sum()), eng.field)
    if cfg.out_csv:
        write_csv(img, cfg.out_csv)
    if cfg.out_pfm:
        write_pfm(img, cfg.out_pfm)
    if cfg.out_png:
        write_png(img, cfg.out_png)
    if cfg.log_path:
        write_convergence_log(log, cfg.log_path)
    if cfg.field_out and eng.field is not None:
        eng.field.save(cfg.field_out)
    return out


@dataclasses.dataclass
class ProbeResult:
    stats: np.ndarray
    seconds: float
    field: Optional[api.GuidingField]


def solve_points(prob: Problem, cfg: RunConfig, points, wpp: int) -> ProbeResult:
    """solve_points (solver.cpp:108-122)."""
    t0 = time.perf_counter()
    eng = Engine(prob, cfg, points)
    for b in range(wpp):
        eng.run_batch(b)
    return ProbeResult(eng.stats(), time.perf_counter() - t0, eng.field)


def mix64(z: int) -> int:
    """Rng::mix (rng.hpp): splitmix64 finaliser."""
    m = (1 << 64) - 1
    z = (z + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def generate_reference(cfg: RunConfig, wpp_ref: int) -> SolutionImage:
    """generate_reference (solver.cpp:169-190): the analytic solution when the
    problem has one, else a long uniform run on an independent seed."""
    prob = load_problem(cfg)
    img = make_image(cfg.width, cfg.height, grid_bbox(cfg, prob))
    if prob.analytic is not None:
        img.cells["mean"] = [prob.analytic(x, y) for x, y in img.cell_centers()]
        img.cells["count"] = 1
        return img
    rc = dataclasses.replace(cfg, mode="uniform", seed=mix64(cfg.seed ^ 0x5EED1EF5))
    img.cells = solve_points(prob, rc, img.cell_centers(), wpp_ref).stats
    return img


@dataclasses.dataclass
class AblationRow:
    mode: str
    relmse: float
    seconds: float
    log: List[LogRow]
    wpp: int = 0


def run_ablation(cfg: RunConfig, modes, reference: SolutionImage) -> List[AblationRow]:
    """run_ablation (solver.cpp:192-232): every mode at equal samples."""
    if not modes:
        raise ValueError("run_ablation: mode list is empty")
    rows = []
    for mode in modes:
        mc = dataclasses.replace(cfg, mode=parse_sampler_mode(mode), out_csv="", out_pfm="", out_png="",
                                 log_path="", field_out="")
        prob = load_problem(mc)
        img = make_image(mc.width, mc.height, grid_bbox(mc, prob))
        eng = Engine(prob, mc, img.cell_centers())
        log = []
        t0 = time.perf_counter()
        for b in range(mc.wpp):
            eng.run_batch(b)
            img.cells = eng.stats()
            log.append(LogRow(b + 1, compute_relmse(img, reference), time.perf_counter() - t0))
        rows.append(AblationRow(mode, log[-1].relmse, log[-1].seconds, log, mc.wpp))
    return rows


def run_equal_time(cfg: RunConfig, modes, reference: SolutionImage, seconds: float,
                   max_wpp: int = 1 << 20) -> List[AblationRow]:
    """Equal-time comparison (the paper's cfg-2 protocol; no reference
    counterpart): every mode runs rounds until its wall time
    reaches `seconds` (the round in flight completes) and reports its relMSE
    and the samples per point it reached."""
    rows = []
    for mode in modes:
        mc = dataclasses.replace(cfg, mode=parse_sampler_mode(mode), out_csv="", out_pfm="", out_png="",
                                 log_path="", field_out="")
        prob = load_problem(mc)
        img = make_image(mc.width, mc.height, grid_bbox(mc, prob))
        eng = Engine(prob, mc, img.cell_centers())
        log = []
        t0 = time.perf_counter()
        b = 0
        while b < max_wpp:
            eng.run_batch(b)
            b += 1
            img.cells = eng.stats()  # synchronises: the clock covers the device work
            el = time.perf_counter() - t0
            log.append(LogRow(b, compute_relmse(img, reference), el))
            if el >= seconds:
                break
        rows.append(AblationRow(mode, log[-1].relmse, log[-1].seconds, log, b))
    return rows
