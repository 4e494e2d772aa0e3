"""paper_1809_07858_b200 — B200-native Shouji pre-alignment filter (arXiv 1809.07858).

Drop-in for the reference's ``prefilter::shouji_filter`` path: the decision for
every pair is computed by hand-written sm_100a kernels (csrc/) behind a C ABI
(include/shouji_b200.h); this package is the host-side mirror of the reference
interface. Importing it loads the compiled extension and fails loudly when it is
missing — there is no CPU fallback.
"""
from .api import (  # noqa: F401
    Context,
    bitvector,
    default_context,
    default_window_width,
    device_count,
    device_error,
    device_pitch,
    empty_sequence_error,
    error,
    filter_decision,
    generate_device,
    illegal_character_error,
    invalid_parameters_error,
    launch_count,
    transfer_bytes,
    length_mismatch_error,
    max_window_width,
    min_window_width,
    out_of_band_error,
    packed_sequence,
    parse_error,
    run_filter,
    seq,
    shouji_filter,
    shouji_filter_batch,
    shouji_filter_device,
    shouji_filter_device_async,
    int_peak,
    profile_stages,
    packed_words,
    pack_planes,
    shouji_filter_packed_batch,
    shouji_filter_packed_device,
    magnet_filter,
    magnet_filter_batch,
    magnet_filter_device,
    nibble_pitch,
    dibit_pitch,
    nplane_pitch,
    host_pack_dibits,
    shouji_filter_dibits_device,
    host_pack_nibbles,
    shouji_filter_nibbles_device,
    threshold_too_large_error,
    unpack_bitmap,
    banded_edit_distance,
    banded_edit_distance_batch,
    pair_dataset,
    load_pairs,
    load_pairs_file,
    generate_pairs,
    write_pairs,
)

__version__ = "0.1.0"
