"""paper_1310_6736_b200 -- B200-native hot path of the salvox 3D salient-region detector.

Drop-in for the reference's exhaustive Kadir-Brady pass, seed-grid detector
(shift / quadrant / octant ascent) and detection selection, computed by
hand-written sm_100a kernels behind the C-ABI in include/salvox_capi.h.
"""
from ._lib import (DET_DTYPE, MAX_DTYPE, Context, SalvoxCudaError, SalvoxError,
                   default_context)
from .api import (DEFAULT_BUDGET, abmsod, abmsod_records, bandwidth_from_moment, dedupe_top_k, detect, detect_batch_device, detect_records,
                  detect_shard, detection_to_dict,
                  exhaustive_debug_hist, kadir_brady_exhaustive, kadir_brady_exhaustive_records,
                  kadir_brady_exhaustive_slab, make_phantom, make_phantom_device, plan_seeds, quadrant_seek,
                  saliency_shift, seek_records, select)

from .api import hu_filter, hu_moments, hu_template_distance, jaccard, rasterize_window
from .api import (ascent_step, bhattacharyya, box_entropy_bits, candidate_histogram, entropy_bits,
                  entropy_nats, mixture_entropy, mixture_entropy_derivative, pdf_difference,
                  shift_step, window_ops)
from .meta_io import load_volume, load_volume_device, save_volume

__version__ = "0.1.0"
