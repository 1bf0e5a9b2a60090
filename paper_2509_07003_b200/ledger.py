"""Byte accounting of collectives (API mirror of spmdsim.comm.CollectiveLedger,
reference comm.py:28-86).

Each record stores the ring-model traffic per participant: 2*S*(P-1)/P for an
all-reduce, S*(P-1)/P for an all-gather or reduce-scatter, with S the full
payload -- the same convention as NCCL-tests bus bandwidth, which bench.py
reports.  Modelled time = traffic x transfer_time_per_byte (latency omitted).
"""

from __future__ import annotations

import csv
import io
from collections import Counter
from fractions import Fraction
from typing import NamedTuple

_RING_FACTOR = {"all_reduce": 2}


def ring_bytes_per_device(collective: str, payload: int, participants: int) -> Fraction:
    if participants <= 1:
        return Fraction(0)
    return Fraction(_RING_FACTOR.get(collective, 1) * payload * (participants - 1), participants)


class LedgerEntry(NamedTuple):
    collective: str
    mesh: str
    dims: str
    payload_bytes: int
    participants: int
    bytes_per_device: Fraction
    modeled_time: Fraction


class CollectiveLedger:
    def __init__(self, transfer_time_per_byte: Fraction = Fraction(1)):
        self.transfer_time_per_byte = transfer_time_per_byte
        self.entries: list[LedgerEntry] = []
        self.counts: Counter = Counter()

    def record(self, collective: str, payload_bytes: int, participants: int, mesh: str = "",
               dims: str = "") -> LedgerEntry:
        traffic = ring_bytes_per_device(collective, int(payload_bytes), int(participants))
        entry = LedgerEntry(collective, mesh, dims, int(payload_bytes), int(participants), traffic,
                            traffic * self.transfer_time_per_byte)
        self.entries.append(entry)
        self.counts[collective] += 1
        return entry

    @property
    def total_bytes(self) -> Fraction:
        return sum((e.bytes_per_device * e.participants for e in self.entries), Fraction(0))

    @property
    def modeled_time(self) -> Fraction:
        return sum((e.modeled_time for e in self.entries), Fraction(0))

    def count(self, collective: str) -> int:
        return self.counts[collective]

    def reset(self):
        self.entries.clear()
        self.counts.clear()

    def to_csv(self) -> str:
        out = io.StringIO()
        writer = csv.writer(out)
        writer.writerow(["collective", "mesh", "dims", "S_bytes", "P", "bytes_per_device", "T_model"])
        writer.writerows([e.collective, e.mesh, e.dims, e.payload_bytes, e.participants,
                          float(e.bytes_per_device), float(e.modeled_time)] for e in self.entries)
        return out.getvalue()
