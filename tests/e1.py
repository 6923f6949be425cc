"""Worked example E1: a hand-checkable 3-mission instance.

Locations on a line x = [0 (base A), 100 (base B), 10, 20, 80, 90];
T_heli = 10|dx|, T_plane = 6|dx| (integer seconds).  v0 = helicopter at A,
v1 = plane at B.  m0: L2->L3 w=1000; m1: L4->L5 w=2000; m2: L3->L2 w=3000,
helicopter-only.  p = 36000, DAY = 86400.
"""
import numpy as np

from paper_2002_11710_b200.instgen import Instance


def e1_instance() -> Instance:
    x = np.array([0, 100, 10, 20, 80, 90], np.int64)
    dx = np.abs(x[:, None] - x[None, :])
    T = np.stack([10 * dx, 6 * dx]).astype(np.int32)
    return Instance(
        travel_s=T, class_is_heli=np.array([1, 0], np.uint8),
        base_location=np.array([0, 1], np.int32), vehicle_base=np.array([0, 1], np.int32),
        vehicle_class=np.array([0, 1], np.int32),
        pickup_loc=np.array([2, 4, 3], np.int32), delivery_loc=np.array([3, 5, 2], np.int32),
        deadline_s=np.array([1000, 2000, 3000], np.int32), heli_only=np.array([0, 0, 1], np.uint8),
        planted_ptr=np.array([0, 3, 3], np.int32), planted_missions=np.array([0, 1, 2], np.int32),
        name="E1")
