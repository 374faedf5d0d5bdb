"""B200-native FairBatching per-iteration scheduling hot path (fbsim drop-in).

Importing the package changes no process state.  Independent simulations run
side by side on their own streams (cluster replicas in `cluster.run_clusters`,
sweeps): with the driver's default 8 hardware work queues, kernels on more
than 8 streams serialise into waves, so entry points that launch many
simulations at once (bench.py, tests/conftest.py) set
CUDA_DEVICE_MAX_CONNECTIONS=32 before the process creates its CUDA context.
"""
