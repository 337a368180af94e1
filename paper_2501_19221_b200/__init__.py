"""paper_2501_19221_b200 -- B200-native batched multi-replica dynamics loop.

Drop-in for the hot path of the reference ``qubokit`` package (arXiv 2501.19221
comparison solvers): ``solve_pa`` (Parallel Annealing) and ``solve_sbm``
(Simulated Bifurcation), plus ``solve_sa`` (simulated annealing, the reference's other
batched-replica solver); QUBO/Ising in, bitstrings + exact energies out.
The loop runs as hand-written sm_100a CUDA kernels behind the C-ABI in
``include/vxq.h`` (``_lib/libvxq.so``); there is no CPU fallback.

    import paper_2501_19221_b200 as vxq
    ss = vxq.solve_pa(model, vxq.PaParams(steps=1000, replicas=1024, seed=0))
    ss.best.energy, vxq.spins_to_bits(ss.best.state)
"""

from .errors import QubokitError, ValidationError
from .model import (IsingModel, QuboModel, as_bits, as_spins, bits_to_spins, sign_pm,
                    spins_to_bits)
from .transforms import qubo_to_ising
from .solvers import (PaParams, SaParams, Sample, SampleSet, SbmParams, default_config,
                      integrate, pa_schedule, params_from_dict, params_to_dict,
                      replica_streams, resolve_c0, resolve_lambda0, run_pa, run_sa, run_sbm,
                      sa_schedule, sbm_schedule, solve_pa, solve_sa, solve_sbm)
from .device import GeneratedModel, clear_cache, energies
from .instance_io import read_instance, write_instance

__version__ = "0.1.0"

__all__ = [
    "QubokitError", "ValidationError", "IsingModel", "QuboModel", "as_bits", "as_spins",
    "bits_to_spins", "sign_pm", "spins_to_bits", "qubo_to_ising", "PaParams", "SbmParams",
    "Sample", "SampleSet", "default_config", "integrate", "params_from_dict", "params_to_dict",
    "replica_streams", "resolve_c0", "resolve_lambda0", "run_pa", "run_sbm", "solve_pa",
    "solve_sbm", "pa_schedule", "sbm_schedule", "clear_cache", "energies", "GeneratedModel",
    "SaParams", "solve_sa", "run_sa", "sa_schedule",
    "read_instance", "write_instance",
]
