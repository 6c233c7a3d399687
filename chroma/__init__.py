"""`chroma` import path for the B200 backend (the reference ships `chroma` as an
implicit namespace package with modules graph, partition, runtime, localcolor,
protocol and verify; each is re-exported here from paper_2107_00075_b200)."""
