"""CPU oracle — TEST INFRASTRUCTURE ONLY (never imported by the product package).

``fvv_oracle`` is the numpy restatement of the reference's edge-server path;
``c_oracle`` binds the plain-C restatement (``c/fvv_oracle.c``) used as the
timed CPU baseline.
"""
