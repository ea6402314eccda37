"""ZipCCL hot path, B200-native (sm_100a).

Drop-in for the reference ``zipcoll`` package API (reference
pkg/src/zipcoll/__init__.py:11-67): the lossless BF16 exponent codec and the
compressed all-gather / all-to-all built on it, with the element work in
hand-written CUDA kernels (libzipccl_b200.so, C-ABI in include/zipccl_b200.h)
and the transfers on NCCL over NVLink or direct NVLink peer reads.
"""

from .bf16 import from_float32, from_float64, measure_sigma, to_float32, to_float64
from .codec import (
    GROUP_SIZE,
    WINDOW_OPT_U,
    CompressedChunk,
    ExponentCodebook,
    codebook_for,
    compress,
    decompress,
    decompress_group,
    derive_codebook,
    optimal_base_exponent,
    static_size_bytes,
    window_coverage,
)
from .container import (
    StaticDynamicSplit,
    parse,
    read_zbf16,
    serialize,
    split_static_dynamic,
    write_zbf16,
)
from .errors import (
    CollectiveError,
    CorruptChunkError,
    CorruptFrameError,
    DegenerateDataError,
    ExtensionMissingError,
    ProfilingError,
    ProtocolError,
    TransportError,
    TransportTimeout,
    UnrepresentableError,
    ZipcollError,
)

__version__ = "0.1.0"


def __getattr__(name):
    # collectives / switcher / transport pull in torch.distributed; load lazily
    import importlib
    for mod in ("collectives", "switcher", "transport"):
        try:
            m = importlib.import_module(f".{mod}", __name__)
        except ModuleNotFoundError:
            continue
        if hasattr(m, name):
            return getattr(m, name)
    raise AttributeError(name)
