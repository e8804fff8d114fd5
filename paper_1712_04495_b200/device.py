"""Simulated device descriptions: the inputs of the simulator that come from
memshare/device.py (`MIB` at :29, `DeviceSpec` at :40-44,
`parse_device_config` at :59-73, `load_device_spec` at :47-56).  Same
schema, same errors."""

from __future__ import annotations

import json
from dataclasses import dataclass

from .errors import ParseError, SchemaError

MIB = 1 << 20


@dataclass(frozen=True)
class DeviceSpec:
    index: int
    name: str
    total_bytes: int

    @property
    def mib(self) -> int:
        return self.total_bytes // MIB


def parse_device_config(doc) -> list[DeviceSpec]:
    """{"devices": [{"name": str, "mib": positive int}, ...]} -> DeviceSpec list."""
    if not isinstance(doc, dict) or not isinstance(doc.get("devices"), list):
        raise SchemaError('expected {"devices": [...]}')
    entries = doc["devices"]
    if not entries:
        raise SchemaError("devices list is empty")
    out = []
    for i, ent in enumerate(entries):
        if not isinstance(ent, dict) or "mib" not in ent:
            raise SchemaError(f"device {i}: expected an object with 'mib'")
        mib = ent["mib"]
        if not isinstance(mib, int) or isinstance(mib, bool) or mib <= 0:
            raise SchemaError(f"device {i}: 'mib' must be a positive integer")
        out.append(DeviceSpec(i, str(ent.get("name", f"sim{i}")), mib * MIB))
    return out


def load_device_spec(path: str) -> list[DeviceSpec]:
    try:
        with open(path) as f:
            doc = json.load(f)
    except (OSError, json.JSONDecodeError) as exc:
        raise ParseError(f"{path}: {exc}") from exc
    return parse_device_config(doc)
