"""B200-native hot path of the Warpspeed data-volume estimator (arXiv 2204.14242).

The product is libwsb200.so (include/ws.h); `ws` is its thin ctypes binding and
`dist` the torch.distributed sharding (one allgather).  Nothing here imports
`oracle/`.
"""
from .ws import (CONFIG_DTYPE, RESULT_DTYPE, Context, WSError, config_array, load_library,  # noqa: F401
                 result_dicts)
