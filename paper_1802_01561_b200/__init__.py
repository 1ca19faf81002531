"""B200-native IMPALA V-trace learner hot path (arxiv 1802.01561, Section 4).

The product is ``libvtrace.so`` (C ABI: ``include/vtrace.h``) built from
``csrc/`` for sm_100a; :mod:`.vtrace` is its thin Python binding and
:mod:`.workload` the seeded synthetic input generator.  There is no CPU
fallback.
"""
from . import workload  # noqa: F401
from .vtrace import (  # noqa: F401
    HeadWorkspace, RmspropWorkspace, VtraceError, Workspace, from_logits, head_loss_and_grad,
    kernel_for, load_library, loss_and_grad, loss_and_grad_from_host, output_layer,
    partials_allreduce, partials_mailbox_bytes, read_device_status, rmsprop_step, status_string,
    tensors_from_workload, version, workspace_bytes)

__version__ = "0.1.0"
