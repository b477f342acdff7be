"""B200-native hybrid-address-space data plane for the devfsim reference
(arXiv 1304.3771, "Paradice").

Public modules mirror the reference's hot-path surface:

* :mod:`.memvirt` -- drop-in for ``devfsim.memvirt`` (page tables,
  translators, ``copy_user_buffer``, hybrid top level) with the data plane
  on sm_100a kernels;
* :mod:`.has` -- drop-in HAS access classes of ``devfsim.backend``
  (``SoftwareHasAccess``, ``HardwareHasAccess``, ``HostNativeAccess``,
  ``GuestProcessRecord``) plus batch copy methods;
* :mod:`.errors` -- the reference's exception types;
* :mod:`.dataplane` -- the batched runtime over ``libpv.so`` (include/pv.h).
"""

__version__ = "0.1.0"
