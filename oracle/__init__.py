"""ORACLE — test infrastructure only.

CPU restatements of the reference hot path used as the checker by tests/,
__graft_entry__.smoke() and bench.py's CPU baseline arm.  The product
package never imports anything from here.
"""
