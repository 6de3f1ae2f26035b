"""paper_2401_13310_b200 — B200-native bulk histogram filling (arXiv 2401.13310).

The compute path is libbhist.so (hand-written sm_100a CUDA behind the C ABI of
include/bhist.h); this package is a thin ctypes binding with the same names.
There is no CPU fallback: if the library is missing or no GPU is present, the
calls raise.
"""
from .bhist import (BH_STRATEGY_AUTO, BH_STRATEGY_CACHE, BH_STRATEGY_EXACT, BH_STRATEGY_GLOBAL, BH_STRATEGY_PRIV,  # noqa: F401
                    BH_STRATEGY_SORT, BH_CONTENT_F64, BH_CONTENT_F32, BH_CONTENT_I32, bh_read_as,
                    BH_DEBUG_SKIP_COPY_WAIT, BH_DEBUG_FIND_BINS_GLOBAL, BH_DEBUG_REQUIRE_JIT, BH_MULTI_PASSES, BH_MULTI_ONE_PASS, BHistError, Histogram, bh_create, bh_destroy, bh_fill,
                    bh_fill_expr, bh_fill_f32, bh_fill_i32, bh_fill_host, bh_fill_host_f32, bh_fill_host_i32, bh_fill_multi, bh_jit_compile_check, bh_pack_multi, bh_packed_size_multi, bh_unpack_multi, bh_find_bins, fill_expr, fill_multi, Program, OPS, bh_get_strategy, bh_info, bh_last_error, bh_launch_count,
                    bh_pack, bh_packed_size, bh_read, bh_reset, bh_set_chunk, bh_set_debug, bh_set_multi_mode, bh_bulk_begin, bh_bulk_submit, bh_bulk_wait, bh_bulk_fill, bh_bulk_end, bh_set_strategy,
                    bh_unpack, bh_version, EXPORTED, lib, library_path)
