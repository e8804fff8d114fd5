"""Exceptions.  The reference's hot path raises only `SchemaError` (from
WorkloadSpec.from_json, memshare/harness.py:115-120; memshare/errors.py:56)
and `ParseError` for unreadable JSON (memshare/errors.py:52); both keep the
reference's names and base class here.  `SgpuError` / `SgpuUnavailable`
report engine failures (no CPU fallback exists)."""


class MemshareError(Exception):
    """Base class (memshare/errors.py MemshareError)."""


class ParseError(MemshareError):
    """A config or workload file is not valid JSON."""


class SchemaError(MemshareError):
    """A config or workload file is valid JSON but violates the schema."""


class SgpuError(MemshareError):
    """A libsgpu entry point returned an error."""


class SgpuUnavailable(SgpuError):
    """libsgpu.so is missing or unusable, or no CUDA device is present."""
