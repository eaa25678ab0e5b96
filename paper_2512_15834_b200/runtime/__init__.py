"""Native runtime: ctypes boundary, paged KV pool, GPU decoder, phase executors."""
