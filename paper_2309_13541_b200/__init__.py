"""B200-native executor for lowered decomposed-MCF all-to-all schedules
(arXiv 2309.13541).  See DESIGN.md.

The drop-in surface mirrors the reference package ``a2aflow``: graphs
(Digraph + generators), schedules (Instruction / ChunkedSchedule / XML) and the
executor slot ``replay_timestep_schedule`` (evaluate.py:56-127).
"""
from .graphs import (Digraph, GraphError, NodeMapping, augment_host_bottleneck,  # noqa: F401
                     all_pairs_distances, distance_sum, gen_gen_kautz,
                     gen_hypercube, gen_torus, load_graph, save_graph)
from .lowering import (collapse_aug_routes, collapse_aug_schedule,  # noqa: F401
                       lower_path_to_steps)
from .schedule import (ChunkedSchedule, Instruction, ScheduleError,  # noqa: F401
                       emit_schedule_xml, parse_schedule_xml)

__version__ = "0.1.0"


def __getattr__(name):
    # the executor needs the native library; import it lazily so the pure
    # host helpers stay usable while it is being built
    if name in ("EvalError", "ExecutorError", "Plan", "replay_timestep_schedule",
                "execute_timestep_schedule", "contiguous_placement"):
        from . import executor
        return getattr(executor, name)
    raise AttributeError(name)
