"""B200-native edge labeling L = T o P (OR-AND semiring) for LTL planning
abstractions -- a drop-in for the reference's labeling path
(ltlgrid::label_all, proj/core/src/label.cpp:150-189).

  label.LabelEngine   load abstraction -> submit grid -> get labels (C ABI)
  label.label_all     one-shot drop-in for ltlgrid::label_all
  (workload.synth     synthetic T / P of the BASELINE configs: not part of the product)
"""
from .label import (CsrBoolMatrix, DensePropMatrix, DomainError, EdgeLabeling, FootprintSpec, LabelEngine,  # noqa: F401
                    LabelMatrix, LtlgError, OccupancyBitset, ScenarioConfig, SweptVolume, generate_scenario,
                    label_all, rasterize_boxes,
                    read_csb1_shape, read_zobv, swept_volume, swept_volume_matrix, to_csr)

__all__ = ["CsrBoolMatrix", "DensePropMatrix", "DomainError", "EdgeLabeling", "FootprintSpec", "LabelEngine", "LabelMatrix",
           "LtlgError", "OccupancyBitset", "ScenarioConfig", "SweptVolume", "generate_scenario", "label_all", "rasterize_boxes", "read_csb1_shape",
           "read_zobv", "swept_volume", "swept_volume_matrix", "to_csr"]
