"""paper_1308_1472_b200 -- B200-native ForestClaw hot path (arXiv 1308.1472).

The product is libfc.so (C ABI in include/fc.h, CUDA for sm_100a); this package is its thin
Python binding.  Build with `python -m paper_1308_1472_b200.build`.
"""
from .fc import (Forest, FcError, forest_for, run, fc_nccl_unique_id, lib, EXPORTS,  # noqa: F401
                 FC_OK, FC_ECFL, FC_ENONFINITE, FC_HOST, FC_DEVICE, FC_ADV_CONST,
                 FC_ADV_EDGEVEL_CAPA, FC_SWE_ROE, FC_EULER_ROE, FC_EULER_HLLE, FC_LIM_NONE, FC_LIM_MINMOD,
                 FC_LIM_MC)
