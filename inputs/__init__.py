"""Seeded synthetic workloads (no method arithmetic). See inputs/configs.py."""
from .configs import (CONFIGS, TTR_CONFIGS, VI_CONFIGS, MdpWorkload, make_reward, Workload, axis_nodes, coarsened, holonomic, make_v0, sub_box)  # noqa: F401
