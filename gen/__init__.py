"""Seeded synthetic inputs for the NRTO inner solve (configs c1-c5).

This package holds NO arithmetic of the method (no costates, no SOC data,
no projections, no solves).  It only produces the *boundary inputs* of one
successive-linearization (SL) iteration -- model Jacobians at a nominal,
constraint gradients and values, the uncertainty-set factor Psi, weights --
exactly the arrays `nrto_setup` consumes (include/nrto.h).  Both the oracle
(oracle/) and the CUDA path (paper_2603_02642_b200/) read these arrays; they
share nothing else.
"""
from .problems import (CONFIGS, make_config, make_instance, make_batch,
                       stack_instances, config_shape)

__all__ = ["CONFIGS", "make_config", "make_instance", "make_batch",
           "stack_instances", "config_shape"]
