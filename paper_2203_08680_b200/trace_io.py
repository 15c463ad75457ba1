"""CSV run traces in the reference's format (trace_io.hpp:18-144).

``CsvTraceWriter`` is a TraceSink: improvement rows are always written,
boundary rows act as a heartbeat (dropped unless ``heartbeat_seconds``
passed since the last row).  Numbers are written like ``std::to_chars``
(shortest round-trip digits, fixed or scientific notation — whichever is
shorter, fixed on a tie), so files are byte-identical to the reference's and
``parse_trace`` reads either back losslessly.
"""
from __future__ import annotations

from decimal import Decimal
from typing import IO, Iterable, List

from .engine import TraceRecord, TraceSink

TRACE_HEADER = "seconds,evaluations,generation,population,fitness"


def format_double(x: float) -> str:
    """std::to_chars(double): shortest round-trip, %f vs %e by length."""
    x = float(x)
    if x != x:
        return "nan"
    if x in (float("inf"), float("-inf")):
        return "inf" if x > 0 else "-inf"
    if x == 0.0:
        return "-0" if str(x).startswith("-") else "0"
    sign, digits, exp = Decimal(repr(x)).normalize().as_tuple()
    d = "".join(map(str, digits))
    point = len(d) + exp  # value = 0.d * 10**point
    if point >= len(d):
        fixed = d + "0" * (point - len(d))
    elif point > 0:
        fixed = d[:point] + "." + d[point:]
    else:
        fixed = "0." + "0" * (-point) + d
    e = point - 1
    sci = d[0] + ("." + d[1:] if len(d) > 1 else "") + "e" + ("-" if e < 0 else "+") + f"{abs(e):02d}"
    body = fixed if len(fixed) <= len(sci) else sci
    return ("-" if sign else "") + body


class CsvTraceWriter(TraceSink):
    """trace_io.hpp:33-76."""

    def __init__(self, out: IO[str], heartbeat_seconds: float = 0.5):
        self.out, self.heartbeat = out, heartbeat_seconds
        self.last_seconds = 0.0
        self.wrote_any = False
        out.write(TRACE_HEADER + "\n")

    def improvement(self, r: TraceRecord):
        self._row(r)

    def boundary(self, r: TraceRecord):
        if self.wrote_any and r.seconds - self.last_seconds < self.heartbeat:
            return
        self._row(r)

    def _row(self, r: TraceRecord):
        self.out.write(f"{format_double(r.seconds)},{format_double(r.evaluations)},{int(r.generation)},"
                       f"{int(r.population)},{format_double(r.fitness)}\n")
        self.out.flush()
        self.last_seconds = r.seconds
        self.wrote_any = True


def parse_trace(lines: Iterable[str]) -> List[TraceRecord]:
    """trace_io.hpp:101-134: header check, 5 fields per row, empty lines skipped."""
    it = iter(lines)
    try:
        head = next(it).rstrip("\n")
    except StopIteration:
        head = None
    if head != TRACE_HEADER:
        raise ValueError("trace: missing or malformed header")
    out = []
    for no, line in enumerate(it, start=2):
        line = line.rstrip("\n")
        if not line:
            continue
        f = line.split(",")
        if len(f) != 5:
            raise ValueError(f"trace: line {no}: expected 5 fields")
        try:
            out.append(TraceRecord(float(f[0]), float(f[1]), int(f[2]), int(f[3]), float(f[4])))
        except ValueError as exc:
            raise ValueError(f"trace: line {no}: bad field ({exc})") from None
    return out


def trace_monotone(records: List[TraceRecord]) -> bool:
    """trace_io.hpp:137-144: wall clock and elitist fitness never go backwards."""
    return all(b.seconds >= a.seconds and b.fitness >= a.fitness for a, b in zip(records, records[1:]))
