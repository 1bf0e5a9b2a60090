"""Collectives over NCCL process groups, byte ledger, bucketing and N-d fusion.

API mirror of spmdsim.comm (reference: /root/reference/pkg/src/spmdsim/
comm.py:1-318).  The reference simulates every device in one process and sums
in ascending rank order; here each process is one rank (one B200) and the
collectives are NCCL calls on per-fiber process groups.  The ledger keeps the
reference's ring byte model (comm.py:45-62), which is also the NCCL-tests
bus-bandwidth convention used by bench.py.
"""

from __future__ import annotations

import csv
import io
from dataclasses import dataclass, field
from fractions import Fraction

DEFAULT_BUCKET_BYTES = 65536


class CommError(ValueError):
    pass


@dataclass
class LedgerEntry:
    collective: str
    mesh: str
    dims: str
    payload_bytes: int
    participants: int
    bytes_per_device: Fraction
    modeled_time: Fraction


@dataclass
class CollectiveLedger:
    """Per-call byte accounting: 2S(P-1)/P for all-reduce, S(P-1)/P for
    all-gather / reduce-scatter (S = full payload)."""

    transfer_time_per_byte: Fraction = Fraction(1)
    entries: list = field(default_factory=list)
    counts: dict = field(default_factory=dict)

    def record(self, collective: str, payload_bytes: int, participants: int, mesh: str = "",
               dims: str = "") -> LedgerEntry:
        P, S = int(participants), int(payload_bytes)
        k = 2 if collective == "all_reduce" else 1
        per_dev = Fraction(k * S * (P - 1), P) if P > 1 else Fraction(0)
        e = LedgerEntry(collective, mesh, dims, S, P, per_dev, per_dev * self.transfer_time_per_byte)
        self.entries.append(e)
        self.counts[collective] = self.counts.get(collective, 0) + 1
        return e

    @property
    def total_bytes(self) -> Fraction:
        return sum((e.bytes_per_device * e.participants for e in self.entries), Fraction(0))

    @property
    def modeled_time(self) -> Fraction:
        return sum((e.modeled_time for e in self.entries), Fraction(0))

    def count(self, collective: str) -> int:
        return self.counts.get(collective, 0)

    def reset(self):
        self.entries.clear()
        self.counts.clear()

    def to_csv(self) -> str:
        buf = io.StringIO()
        w = csv.writer(buf)
        w.writerow(["collective", "mesh", "dims", "S_bytes", "P", "bytes_per_device", "T_model"])
        for e in self.entries:
            w.writerow([e.collective, e.mesh, e.dims, e.payload_bytes, e.participants,
                        float(e.bytes_per_device), float(e.modeled_time)])
        return buf.getvalue()
