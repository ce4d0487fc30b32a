"""Drop-in binding of the reference package `vexsort` to the B200 C ABI
(the stub INTEGRATION.md describes, as code).  See _kernels_b200.py."""
