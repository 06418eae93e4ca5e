"""Quantity parsing for link-profile files.

Mirrors the conventions of the reference's ``linkstripe.units``
(`pkg/src/linkstripe/units.py:58-99`): byte sizes take *binary*
prefixes (``"4M"`` is 4 MiB, nccl-tests style), rates take *decimal*
prefixes (``"64 GB/s"`` is 64e9 B/s) and a lowercase ``b`` in a rate
means bits (``"400 Gb/s"`` is 50e9 B/s).
"""

from __future__ import annotations

import re

__all__ = ["parse_size", "parse_bandwidth", "parse_time", "gbps", "format_size"]

_QUANTITY = re.compile(r"^\s*([0-9]*\.?[0-9]+(?:[eE][-+]?[0-9]+)?)\s*(\S*)\s*$")

_BINARY = {"": 0, "B": 0, "K": 10, "KB": 10, "KIB": 10, "M": 20, "MB": 20, "MIB": 20,
           "G": 30, "GB": 30, "GIB": 30}
_DECIMAL = {"": 0, "K": 3, "M": 6, "G": 9, "T": 12}
_SECONDS = {"S": 1.0, "MS": 1e-3, "US": 1e-6, "NS": 1e-9}


def _number_and_unit(text) -> tuple[float, str]:
    match = _QUANTITY.match(str(text))
    if match is None:
        raise ValueError(f"cannot parse quantity: {text!r}")
    return float(match.group(1)), match.group(2)


def parse_size(text) -> int:
    """Byte count: ``"256M"``, ``"4MiB"``, ``1048576`` (`units.py:58-66`)."""
    if isinstance(text, (int, float)):
        return int(text)
    value, unit = _number_and_unit(text)
    shift = _BINARY.get(unit.upper())
    if shift is None:
        raise ValueError(f"unknown size unit {unit!r} in {text!r}")
    return int(round(value * (1 << shift)))


def parse_bandwidth(text) -> float:
    """Rate in bytes/s; ``b`` (bits) vs ``B`` (bytes) matters (`units.py:69-85`)."""
    if isinstance(text, (int, float)):
        return float(text)
    value, unit = _number_and_unit(text)
    if not unit:
        return value
    if "/" not in unit:
        raise ValueError(f"unknown bandwidth unit {unit!r} in {text!r}")
    head, tail = unit.split("/", 1)
    if tail.upper() != "S" or not head or head[-1] not in "bB":
        raise ValueError(f"unknown bandwidth unit {unit!r} in {text!r}")
    bits = head[-1] == "b"
    exponent = _DECIMAL.get(head[:-1].upper())
    if exponent is None or (exponent == 0 and head[:-1]):
        raise ValueError(f"unknown bandwidth unit {unit!r} in {text!r}")
    rate = value * (10.0 ** exponent) if exponent else value
    return rate / 8 if bits else rate


def parse_time(text) -> float:
    """Duration in seconds: ``"5us"``, ``"1.5 ms"`` (`units.py:88-99`)."""
    if isinstance(text, (int, float)):
        return float(text)
    value, unit = _number_and_unit(text)
    if not unit:
        return value
    key = unit.replace("µ", "u").replace("μ", "u").upper()
    if key not in _SECONDS:
        raise ValueError(f"unknown time unit {unit!r} in {text!r}")
    return value * _SECONDS[key]


def gbps(bytes_per_second: float) -> float:
    return bytes_per_second / 1e9


def format_size(n_bytes: int) -> str:
    for suffix, shift in (("G", 30), ("M", 20), ("K", 10)):
        unit = 1 << shift
        if n_bytes >= unit and n_bytes % unit == 0:
            return f"{n_bytes // unit}{suffix}"
    return str(n_bytes)
