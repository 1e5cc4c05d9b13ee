"""Exception type mirroring the reference's ``ilsim::Error`` (common.hpp:12-15)
and the Python binding's ``ilsim.IlsimError`` (bindings/module.cpp:209)."""


class IlsimError(RuntimeError):
    pass
