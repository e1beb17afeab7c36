"""B200-native bucket-elimination backend for QAOA tensor-network simulation
(arxiv 2106.15740, "Importance of Diagonal Gates in Tensor Network
Simulations").

Drop-in for the contraction path of the reference package `qtnsim`
(/root/reference/pkg/src/qtnsim): the names re-exported here mirror
qtnsim/__init__.py:9-74 for everything on that path, the contraction runs in
hand-written sm_100a kernels behind a C ABI (include/qtn_b200.h), and the
energy driver / light-cone builder the north star asks for are added.
"""

from . import _native  # noqa: F401  (fails loudly if the library is missing)
from .circuit import (Circuit, Gate, GateKind, ProblemGraph, QaoaParams,
                      build_qaoa_maxcut_circuit, gate_matrix, is_diagonal)
from .contraction import (DEFAULT_MIXED_RANK, DEFAULT_RANK_CAP, ContractionPlan,
                          RankCapExceeded, contract, contract_many)
from .energy import (EnergyPlan, compile_jobs, energy_expectation, plan_edges, rank_shard,
                     shard_edges)
from .lightcone import (EnergyTemplate, build_edge_lightcone_circuit, build_energy_network,
                        edge_lightcone_gates, energy_template)
from .network import (LineGraph, NetworkMode, Tensor, TensorNetwork, circuit_to_network,
                      line_graph, network_stats, sliced_tensors)
from .ordering import (ContractionOrder, CostReport, contraction_width, greedy_order,
                       rgreedy_order)
from .pipeline import (MODE_ORDER, MODES, PipelineMode, build_circuit, build_line_graph,
                       build_network, default_angles, get_mode, random_regular_graph,
                       seeded_angles)

__version__ = "0.1.0"
