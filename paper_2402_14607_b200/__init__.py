"""B200-native block-wise two-source extractor (arXiv 2402.14607).

Drop-in for the hot path of the reference package ``blockext``: the same
extractor API (extract_eq, extract_neq, Extraction, ext_ip, run_parallel, the
GF(2^q) contexts, plans, reports and the sample generator/packer), computed by
hand-written sm_100a kernels (include/blockext_b200.h).  There is no CPU
fallback: without the built library every compute call raises
ExtensionMissingError.
"""
from .errors import (CapacityError, DeviceError, DivergenceError, ExtensionMissingError,
                     InfeasibleError, TruncatedSourceError, UncertifiableError,
                     UnsupportedRateError, VerificationError)
from .extractor import (BlockCursor, BlockPair, BlockProcessingError, Extraction, OutputChunk,
                        ext_ip, extract_eq, extract_neq, run_parallel)
from .gf2q import (MAX_FIELD_BITS, MODULUS_EXPONENTS, GFContext, field, gf_add, gf_mul,
                   is_irreducible, modulus_int)
from .params import (EqPlan, NeqPlan, error_bound_block, error_bound_eq, error_bound_neq,
                     extraction_rate, plan_eq, plan_neq)
from .report import ExtractionReport, plan_from_text, plan_to_text
from .sources import SourceModel, file_source, generate, iid_biased, iid_table, markov
from .verify import (BiasReport, DistanceReport, check_extractor_distance,
                     check_first_bit_bijection, check_hadamard, check_one_bit_bias,
                     check_xor_lemma_instance, hadamard_instances)

__version__ = "0.1.0"
