"""paper_1105_4424_b200 — B200-native Array-OL repetitive-task engine (drop-in for gmodelc's executor).

The hot path of arXiv 1105.4424's Gaspard2/MARTE flow: each point of a
repetition space gathers its input pattern through a tiler, runs an
elementary task and scatters its output pattern.  Python mirrors the
reference's model / schedule / operator-registry API
(/root/reference/pkg/src/gmodelc/) and hands device pointers to
hand-written sm_100a CUDA kernels in libaolb200.so through a C ABI
(include/aol_b200.h).  There is no CPU fallback.
"""

from .intrinsics import (INTRINSICS, IntrinsicShapeMismatch, IntrinsicSpec, PortSpec,  # noqa: F401
                         UnknownIntrinsic, check_task_signature, register_into)
from .model import (AllocKind, AllocationLink, Component, ComponentKind, Connector, DataType,  # noqa: F401
                    Direction, FlowPort, HwStereotype, MemoryRole, Model, PartInstance, Shape,
                    StereotypeKind, UntilCondition)
from .partition import (DeviceStep, HostOp, KernelLaunch, LoopStep, Schedule, WorkRange,  # noqa: F401
                        build_schedule, derive_launch_config, partition_equally)
from .tiler import BoundTiler, Tiler, TilerError  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):
    # the executor imports torch; keep `import paper_1105_4424_b200` light
    if name in ("execute_schedule", "Executor", "ExecutionResult", "MissingBinding"):
        from . import executor
        return getattr(executor, name)
    raise AttributeError(name)
