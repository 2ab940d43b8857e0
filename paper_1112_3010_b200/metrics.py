"""Error aggregates of the experiment protocols (R/metrics.py:46-72, 75-90).

percentage_error: 100 |computed - exact| / exact over the nodes with
exact > 0 (`mean`, `maximum`), and the protocol normalisation `paper_mean`
(the same sum divided by the total node count).  Report carries the rows and
the configuration that produced them.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np

from .errors import ValidationError
from .grid import ScalarField


@dataclass(frozen=True)
class ErrorStats:
    mean: float
    maximum: float
    paper_mean: float
    included: int
    total: int
    per_node: ScalarField


def percentage_error(computed: ScalarField, exact: ScalarField) -> ErrorStats:
    if computed.grid != exact.grid:
        raise ValidationError("fields live on different grids")
    c = np.asarray(computed.values, dtype=np.float64)
    e = np.asarray(exact.values, dtype=np.float64)
    inc = e > 0.0
    if not inc.any():
        raise ValidationError("every exact value is zero; nothing to compare")
    pct = np.zeros_like(e)
    pct[inc] = 100.0 * np.abs(c[inc] - e[inc]) / e[inc]
    return ErrorStats(mean=float(pct[inc].mean()), maximum=float(pct[inc].max()),
                      paper_mean=float(pct[inc].sum() / e.size), included=int(inc.sum()), total=int(e.size),
                      per_node=ScalarField(exact.grid, pct))


@dataclass
class Report:
    name: str
    config: dict
    rows: list = field(default_factory=list)

    def to_json(self) -> str:
        return json.dumps({"experiment": self.name, "config": self.config, "rows": self.rows}, sort_keys=True,
                          indent=2) + "\n"
