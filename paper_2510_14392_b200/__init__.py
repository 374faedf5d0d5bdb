"""B200-native FairBatching per-iteration scheduling hot path (fbsim drop-in)."""
import os as _os

# Independent simulations run side by side on their own streams (sweeps,
# cluster replicas): with the default 8 hardware work queues, kernels on more
# than 8 streams serialise into waves.  Takes effect if set before the
# process creates its CUDA context.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
