"""Exception hierarchy mirroring the reference's (ucores/errors.hpp:8-115).

Only the classes the mapCL / mapCLPartition / reduceCL path can raise are
mirrored; names and meanings follow the reference so callers catch the same
types.
"""


class Error(RuntimeError):
    """ucores::Error (errors.hpp:9-12): base of every library error."""


class ElementKindError(Error):
    """errors.hpp:27-29: element variant mismatch."""


class MixedElementVariants(Error):
    """errors.hpp:30-34: a partition mixes element variants (concat)."""


class InvalidPartitionCount(Error):
    """errors.hpp:14-17: create_dataset with num_partitions < 1."""


class UnknownKernel(Error):
    """errors.hpp:41-44: no kernel registered under that name."""


class ArityMismatch(Error):
    """errors.hpp:45-48: unary kernel used where binary expected or vice versa."""


class DuplicateKernelName(Error):
    """errors.hpp:37-40."""


class KernelPanic(Error):
    """errors.hpp:55-63: failure inside a kernel phase; carries the phase."""

    def __init__(self, phase: str, detail: str):
        super().__init__(f"kernel panic in {phase}: {detail}")
        self.phase = phase


class PeerExchangeError(KernelPanic):
    """A sharded reduce_cl's NVLink exchange timed out: a peer rank never
    published its partials (the affected launch wrote NaN / -1, not a
    plausible value). Every later launch on that exchange raises this until
    all ranks call MapReducePipeline.reset_exchange()."""


class EmptyDataset(Error):
    """errors.hpp:80-83: reduce_cl over zero elements."""


class JobFailed(Error):
    """errors.hpp:84-87: a task failed on every attempt (max_retries + 1)."""


class LengthMismatch(Error):
    """errors.hpp:112-115: reduced vectors differ in length."""


class DeviceUnavailable(Error):
    """No usable sm_100 device / native library: the product has no CPU fallback."""
