"""Run configuration: drop-in mirrors of the reference dataclasses.

EmbeddingConfig   engine.py:30-84     (defaults nn=3, rn=1, c=0.1, 2500 iters)
IntegratorParams  optim.py:15-56      (a=0.99, b=0.002, tau=1e-3*M, gamma 1.1/0.9)
OptimizerParams   optim.py:59-68      (alpha per kind, beta, gamma_v/s, rho, eps)

Instances of the reference's own classes are accepted wherever these are
(duck typing on the field names); `resolve_optimizer` turns either into the
C struct the device consumes.
"""

import warnings
from dataclasses import asdict, dataclass, field, fields

from . import _lib
from .errors import InvalidArgumentError

OPTIMIZER_KINDS = ("force-directed", "sgd", "momentum", "nesterov", "adam", "adadelta")
DISTANCE_MODES = ("binary", "euclidean")
DEFAULT_ALPHA = {"sgd": 0.1, "momentum": 0.02, "nesterov": 0.02, "adam": 0.05, "adadelta": 1.0}


@dataclass
class IntegratorParams:
    """Force-directed constants: delta <- a*delta + b*force (optim.py:15-56)."""

    a: float = 0.99
    b: float = 0.002
    tau: float | None = None
    gamma1: float = 1.1
    gamma2: float = 0.9
    auto_adapt: bool = True
    lam: float | None = None
    dt: float | None = None
    k_nn: float | None = None

    def __post_init__(self):
        if not 0.0 <= self.a <= 1.0:
            raise InvalidArgumentError(f"a must be in [0, 1], got {self.a}")
        if not self.b > 0.0:
            raise InvalidArgumentError(f"b must be positive, got {self.b}")
        if not (self.gamma1 > 1.0 and 0.0 < self.gamma2 < 1.0):
            raise InvalidArgumentError("need gamma1 > 1 and gamma2 in (0, 1)")

    @classmethod
    def from_physics(cls, lam, dt, k_nn, **kwargs):
        """a/b = (1 - lam dt/2) / (2 k_nn dt) (optim.py:42-53)."""
        if dt <= 0 or k_nn <= 0:
            raise InvalidArgumentError("dt and k_nn must be positive")
        half = lam * dt / 2.0
        return cls(a=(1.0 - half) / (1.0 + half), b=2.0 * k_nn * dt / (1.0 + half),
                   lam=lam, dt=dt, k_nn=k_nn, **kwargs)

    def tau_for(self, m):
        return self.tau if self.tau is not None else 1e-3 * m


@dataclass
class OptimizerParams:
    """Knobs of the gradient optimizers (optim.py:59-68)."""

    alpha: float | None = None
    beta: float = 0.9
    gamma_v: float = 0.9
    gamma_s: float = 0.999
    rho: float = 0.95
    eps: float = 1e-8


@dataclass
class EmbeddingConfig:
    """Everything a run needs besides the graph (engine.py:30-84)."""

    nn: int = 3
    rn: int = 1
    c: float = 0.1
    distance_mode: str = "binary"
    iterations: int = 2500
    l1_final_steps: int = 0
    rnn_final_steps: int = 0
    optimizer: str = "force-directed"
    seed: int = 0
    target_dim: int = 2
    rn_resample_period: int = 0
    graph_metric: str = "euclidean"
    normalize_targets: bool = True
    integrator: IntegratorParams = field(default_factory=IntegratorParams)
    opt: OptimizerParams = field(default_factory=OptimizerParams)

    def __post_init__(self):
        checks = (
            (self.nn >= 1 and self.rn >= 1, "nn and rn must be >= 1"),
            (0.0 < self.c < 1.0, f"c must be in (0, 1), got {self.c}"),
            (self.target_dim in (2, 3), "target_dim must be 2 or 3"),
            (self.iterations >= 0, "iterations must be >= 0"),
            (self.l1_final_steps >= 0 and self.rnn_final_steps >= 0,
             "phase step counts must be >= 0"),
            (max(self.l1_final_steps, self.rnn_final_steps) <= self.iterations,
             "final phases cannot exceed total iterations"),
            (self.optimizer in OPTIMIZER_KINDS, f"unknown optimizer {self.optimizer!r}"),
            (self.distance_mode in DISTANCE_MODES,
             f"unknown distance mode {self.distance_mode!r}"),
            (self.rn_resample_period >= 0, "rn_resample_period must be >= 0"),
        )
        for ok, msg in checks:
            if not ok:
                raise InvalidArgumentError(msg)
        if self.nn < self.rn:
            warnings.warn(f"nn={self.nn} < rn={self.rn}: long-range forces may dominate",
                          stacklevel=2)
        if isinstance(self.integrator, dict):
            self.integrator = IntegratorParams(**self.integrator)
        if isinstance(self.opt, dict):
            self.opt = OptimizerParams(**self.opt)

    def to_dict(self):
        return asdict(self)

    @classmethod
    def from_dict(cls, payload):
        return cls(**payload)


def coerce_config(config):
    """Accept this package's config, the reference's, or None."""
    if config is None:
        return EmbeddingConfig()
    if isinstance(config, EmbeddingConfig):
        return config
    return config  # reference EmbeddingConfig: same field names (duck typed)


def resolve_optimizer(kind, m, integrator=None, opt=None):
    """Build the ivhd_optimizer_params struct for `kind` (make_optimizer,
    optim.py:249-256, with the per-kind alpha defaults optim.py:71-77)."""
    if kind not in OPTIMIZER_KINDS:
        raise InvalidArgumentError(f"unknown optimizer {kind!r}; choose from {OPTIMIZER_KINDS}")
    ip = integrator if integrator is not None else IntegratorParams()
    op = opt if opt is not None else OptimizerParams()
    p = _lib.OptimizerParams()
    p.kind = _lib.OPT_KIND[kind]
    p.auto_adapt = int(bool(ip.auto_adapt))
    p.a = float(ip.a)
    p.tau = float(ip.tau if ip.tau is not None else 1e-3 * m)
    p.gamma1 = float(ip.gamma1)
    p.gamma2 = float(ip.gamma2)
    p.beta = float(op.beta)
    p.gamma_v = float(op.gamma_v)
    p.gamma_s = float(op.gamma_s)
    p.rho = float(op.rho)
    p.eps = float(op.eps)
    if kind == "force-directed":
        p.step = float(ip.b)
    else:
        p.step = float(op.alpha if op.alpha is not None else DEFAULT_ALPHA[kind])
    return p


def config_fields():
    return [f.name for f in fields(EmbeddingConfig)]
