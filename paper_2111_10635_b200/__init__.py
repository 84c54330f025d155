"""B200-native plan evaluator for the HeterPS scheduler (arXiv 2111.10635)."""
from .errors import (ConfigError, InfeasibleError, InvariantError, NativeUnavailableError,
                     NumericError, ParseError, PlanValidationError, SchedulerError)
from .model import (CostReport, JobParams, LayerSpec, ModelGraph, ProvisionerConfig,
                    ProvisioningPlan, ResourceCatalog, ResourceType, ScoredPlan,
                    SchedulingPlan, Stage, penalty_cost)
from .graphio import (catalog_with_gpu_variants, load_catalog, load_fixture, load_model_graph,
                      resize_model, save_catalog, save_model_graph, simulate_type_variants)

__version__ = "0.1.0"
