"""B200-native threshold / symmetric queries over bitmaps.

A drop-in, GPU-backed replacement for the hot path of the reference package
``bitquorum`` (Kaser & Lemire, *Threshold and Symmetric Functions Over
Bitmaps*): the threshold theta(T; B_1..B_N) and arbitrary symmetric functions
of the per-position count over N bitmaps, uncompressed or EWAH-style RLE.

Python entry points (reference names and signatures) are in :mod:`.api`; the
device engine (prepared queries, host streaming) in :mod:`.engine`; the
word-range multi-GPU partitioner in :mod:`.shard`; the C ABI underneath is
``include/bq.h`` / ``libbq.so``.
"""

from .api import (
    DEFAULT_BUDGET_BYTES,
    CircuitLibrary,
    CompiledProgram,
    and_,
    andnot,
    binary_op,
    not_,
    or_,
    xor,
    compile_program,
    execute,
    execute_horizontal,
    cdom_symmetric,
    dirty_segment_solver,
    cdom_threshold,
    compress,
    compress_device,
    compress_words,
    counter_width,
    csv_op_count,
    csv_threshold,
    decompress,
    looped_op_count,
    looped_threshold,
    scan_count,
    scan_count_symmetric,
    symmetric,
    threshold,
    to_device,
    weight_bits,
    wide_and,
    wide_or,
)
from .bitmaps import DeviceBitmap, DeviceRleBitmap, RleBitmap, UncompressedBitmap
from .engine import RleQuery, ThresholdQuery, release_cached_memory, sweep_host
from .errors import (
    BitquorumError,
    CorrectnessError,
    DeviceError,
    ExtensionMissing,
    FormatError,
    InputError,
    NoCoveringCircuit,
    ResourceError,
)
from .serial import dumps_bitmap, loads_bitmap_device, read_bitmap_device, write_bitmap
from .similarity import DeviceDataset, SimilarityQuery, make_similarity
from .spec import SymmetricSpec
from . import circuits
from .circuits import (
    BitProgram,
    Circuit,
    PaddingPlan,
    build_sideways_sum,
    build_sop,
    build_sorter,
    build_tree_adder,
    compile_circuit,
    dumps_program,
    loads_program,
    optimize,
    plan_padding,
)

__version__ = "0.1.0"
