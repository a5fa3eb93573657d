"""B200-native (sm_100a) SpargeAttn hot path (arXiv 2502.18137).

    paper_2502_18137_b200.sparge   -- Python binding of libsparge.so (C ABI,
                                      include/sparge.h); imports fail loudly
                                      when the library is not built
    paper_2502_18137_b200.inputs   -- seeded synthetic workload generators
    paper_2502_18137_b200.build    -- nvcc build of libsparge.so (sm_100a)
"""
