"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds ONLY random-number recipes (tables, tasks, cost-model
weights).  It contains none of the method's arithmetic (no featurisation, no
MLP forward, no search); see DESIGN.md "Input recipe".
"""
from .synth import (  # noqa: F401
    CONFIGS,
    Task,
    Weights,
    gen_task,
    gen_tasks,
    gen_weights,
    gen_plans,
)
