"""B200-native deep-potential force evaluation (arXiv 2602.02234 hot path).

Product = libhmdp.so (CUDA sm_100a kernels + C-ABI, include/hmdp.h).  This
package is the host-side mirror of the reference's C++ NN force-provider API
(halomd::nn, /root/reference/proj/include/halomd/nn/) over that C-ABI.
"""
from .nn import (ForceProvider, ModelFamily, NnCounters, NnInput, NnModel, NnOutput, Precision,
                 SimBox, build_input_periodic, context_for, Context, descriptors, evaluate,
                 load_model, make_dp_model, make_model, model_from_json, model_to_json, save_model,
                 switch_derivative, switch_value)
from .synthetic import PAPER_SYSTEMS, generate_synthetic_system, replicate

__all__ = [
    "ForceProvider", "ModelFamily", "NnCounters", "NnInput", "NnModel", "NnOutput", "Precision",
    "SimBox", "build_input_periodic", "context_for", "Context", "descriptors", "evaluate",
    "load_model", "make_dp_model", "make_model", "model_from_json", "model_to_json", "save_model",
    "switch_derivative", "switch_value", "PAPER_SYSTEMS", "generate_synthetic_system", "replicate",
]
