"""B200-native REINFORCE device-placement hot path (arXiv 1706.04972).

Drop-in for the reference package ``devplace`` on its hot path: the graph
input model, the placement scorer (simulator), the seq2seq policy and the
REINFORCE trainer keep the reference names and signatures; the work runs in
hand-written sm_100a CUDA kernels behind the C-ABI in include/devplace_b200.h.
"""

from . import graph, simulator  # noqa: F401
from .graph import (ComputationGraph, CycleError, Edge, GraphError, Group, GroupedGraph,  # noqa: F401
                    GroupEdge, Operation, coalesce_sole_consumers, singleton_groups, topo_order)
from .simulator import (INFEASIBLE, Device, DeviceTopology, NoiseSpec, SimReport,  # noqa: F401
                        TopologyError, check_memory, default_topology, measure, simulate,
                        simulate_batch)

from . import policy, trainer  # noqa: F401,E402
from .policy import (EmbeddingSpec, GroupFeatures, PolicyParams, SampledPlacement,  # noqa: F401,E402
                     embed_groups, forward_sample, grad_log_prob, load_checkpoint, log_prob_of,
                     sample_batch, save_checkpoint, step_distributions)
from .trainer import (BaselineState, LogRow, ParameterStore, RewardSpec, TrainerConfig,  # noqa: F401,E402
                      TrainResult, apply_adam, log_to_csv, reinforce_update, reward_of, run_controller,
                      suggest_failing_signal, train, train_many)

from . import baselines  # noqa: F401,E402
from .baselines import (NoFeasiblePlacement, SearchSpaceTooLarge, brute_force,  # noqa: F401,E402
                        place_random_search, place_single)

__version__ = "0.1.0"
