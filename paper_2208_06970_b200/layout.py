"""Aggregate blob record (the part of the reference's ``lrcvt.layout`` that
the aggregation path emits, layout.py:27-65). The .lrcvt file writer/reader
is out of scope for this build."""

from __future__ import annotations

import json
from dataclasses import dataclass

from .stats import MomentAggregate

AGG_MOMENTS = 1
AGG_JSON = 2
SCOPES = ("region", "component", "layer")


@dataclass
class AggregateBlob:
    scope: str  # region | component | layer
    scope_id: int
    kind: int
    payload: bytes

    @classmethod
    def moments(cls, scope: str, scope_id: int, agg: MomentAggregate) -> "AggregateBlob":
        return cls(scope, scope_id, AGG_MOMENTS, json.dumps(agg.to_dict()).encode())

    def as_moments(self) -> MomentAggregate:
        if self.kind != AGG_MOMENTS:
            raise ValueError(f"blob kind {self.kind} is not a moment aggregate")
        return MomentAggregate.from_dict(json.loads(self.payload.decode()))
