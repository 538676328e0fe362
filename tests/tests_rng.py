"""mt19937_64 draws of the reference tests (rng.hpp), via the oracle's C
restatement, to reproduce their parameter sequences."""
import ctypes as C

import oracle as O


class Rng:
    def __init__(self, seed: int):
        self.lib = O._oracle_lib()
        self.lib.so_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
        self.lib.so_rng_next.restype = C.c_uint64
        self.lib.so_rng_next.argtypes = [C.c_void_p]
        self.lib.so_rng_below.restype = C.c_uint64
        self.lib.so_rng_below.argtypes = [C.c_void_p, C.c_uint64]
        self.buf = C.create_string_buffer(312 * 8 + 8)
        self.lib.so_rng_seed(self.buf, seed)

    def next_u64(self) -> int:
        return int(self.lib.so_rng_next(self.buf))

    def below(self, n: int) -> int:
        return int(self.lib.so_rng_below(self.buf, n))
