"""Error types for the B200 offload engine.

Same class names and machine codes as the reference's ``moesim.errors``
(errors.py:10-84) so callers that catch ``SimError`` subclasses or switch on
``.code`` keep working.  The C-ABI returns integer status codes; ``raise_for``
maps them onto these classes (see include/fate_b200.h).
"""

from __future__ import annotations


class SimError(Exception):
    code = "SIM_ERROR"

    def __init__(self, message: str, code: str | None = None):
        super().__init__(message)
        if code is not None:
            self.code = code


def _kind(name: str, code: str, doc: str) -> type:
    return type(name, (SimError,), {"code": code, "__doc__": doc})


InvalidConfig = _kind("InvalidConfig", "INVALID_CONFIG", "A config, policy or knob violates an invariant.")
TraceIOError = _kind("TraceIOError", "TRACE_IO", "A trace file could not be read or written.")
SchemaError = _kind("SchemaError", "TRACE_SCHEMA", "A trace record is malformed or inconsistent.")
TraceMismatch = _kind("TraceMismatch", "TRACE_MISMATCH", "Trace geometry does not match the model config.")
DegenerateGen = _kind("DegenerateGen", "DEGENERATE_GEN", "Trace-generation similarity targets are unsatisfiable.")
ZeroVector = _kind("ZeroVector", "ZERO_VECTOR", "Cosine similarity of a zero vector.")
MissingProbes = _kind("MissingProbes", "MISSING_PROBES", "A trace lacks the probe hidden states a step needs.")
BudgetTooSmall = _kind("BudgetTooSmall", "BUDGET_TOO_SMALL", "Memory budget is below the dense footprint.")
NoAccesses = _kind("NoAccesses", "NO_ACCESSES", "Hit rate requested over zero accesses.")
CorruptCodes = _kind("CorruptCodes", "CORRUPT_CODES", "Quantized codes outside the representable range.")
NoFeasibleP = _kind("NoFeasibleP", "NO_FEASIBLE_P", "No INT2 fraction meets the loss tolerance.")


class DeviceError(SimError):
    """The CUDA extension failed (launch error, OOM, missing library or GPU)."""

    code = "DEVICE_ERROR"


# C-ABI status codes (include/fate_b200.h, FATE_E*) -> exception classes.
_STATUS = {
    1: InvalidConfig,
    2: TraceMismatch,
    3: BudgetTooSmall,
    4: CorruptCodes,
    5: DeviceError,
    6: DeviceError,
}


def raise_for(status: int, what: str, detail: str = "") -> None:
    if status == 0:
        return
    cls = _STATUS.get(status, DeviceError)
    raise cls(f"{what} failed with status {status}{': ' + detail if detail else ''}")
