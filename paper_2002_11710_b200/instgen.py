"""Seeded synthetic air-EMS instances shaped like the paper's workloads.

INPUT GENERATION ONLY.  This module is the one piece shared by the CPU oracle
(`oracle/`) and the CUDA path: it produces the *inputs* (locations, an integer
second travel-time matrix, vehicles, missions with deadlines) and a planted
feasible start schedule.  It contains none of the method's arithmetic (no
objective, no feasibility check, no move evaluation, no search).

Paper sources for the shapes:
  * bases P (planes) / H (helicopters), each a <id, speed, lat, lon> tuple
    (§3, lines 44-66); 12 vehicles = 8 helicopters + 4 planes (§5);
  * missions <id, pickup lat/lon, delivery lat/lon, rho> (§3),
    deadlines "randomly generated ... within a 24 hour period" (§5);
  * speeds 300 km/h (helicopter) / 500 km/h (plane) (§3);
  * Haversine travel time, Eq. e1 (§3), r = 6371.0 km (reading #11,
    DESIGN.md) and rounded to integer seconds (BASELINE.json north_star).

Recipe: facilities and base sites are drawn in a
region (Ontario-like box for C1-C3, a ~300 km regional cluster for C4, a 60 km
disaster zone for C5); vehicles go to bases round-robin by class; missions are
*planted* on random vehicles, each pickup drawn among the K facilities nearest
the vehicle's base and each delivery among the K nearest the pickup; the
deadline is the planted arrival plus uniform slack, so the planted routes are
feasible by construction (flight <= 0.9 p, return <= 24 h).  Mission ids are
shuffled at the end.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

EARTH_RADIUS_KM = 6371.0          # reading #11 (paper leaves r unstated)
SPEED_KMH = (300.0, 500.0)        # class 0 = helicopter, class 1 = plane
CLASS_IS_HELI = (1, 0)
FLIGHT_LIMIT_S = 36000            # p = 10 h
DAY_S = 86400                     # 24 h return limit
SEED_BASE = 2002117100            # instance seed = SEED_BASE + config number

# Ontario-like cluster centres (synthetic stand-ins for the dense south + a few
# northern hubs; the paper's coordinates are unpublished).
_ONTARIO_BOX = (42.0, 50.0, -95.0, -74.0)
_ONTARIO_SOUTH = [(43.70, -79.40), (45.40, -75.70), (42.30, -83.00), (43.25, -79.87),
                  (44.23, -76.48), (42.98, -81.25), (44.40, -79.70)]
_ONTARIO_NORTH = [(46.50, -81.00), (48.40, -89.25), (49.77, -94.49), (46.31, -79.46)]


@dataclasses.dataclass
class Config:
    name: str
    n_missions: int
    n_heli_vehicles: int
    n_plane_vehicles: int
    n_heli_bases: int
    n_plane_bases: int
    n_facilities: int
    region: str                  # "ontario" | "regional" | "disaster"
    locality: int                # K nearest facilities used when planting
    max_iters: int
    tenure: int
    n_runs: int = 1
    kick: int = 0

    @property
    def n_vehicles(self) -> int:
        return self.n_heli_vehicles + self.n_plane_vehicles

    @property
    def n_bases(self) -> int:
        return self.n_heli_bases + self.n_plane_bases


# BASELINE.json "configs", resolved in SURVEY.md §8.0 (daggered values are proposals).
CONFIGS = {
    "tiny": Config("tiny", 8, 2, 1, 1, 1, 10, "ontario", 6, 200, 5),
    "ontario": Config("ontario", 60, 13, 7, 8, 4, 60, "ontario", 8, 5000, 10),
    "batched": Config("batched", 100, 13, 7, 8, 4, 60, "ontario", 8, 1000, 10, n_runs=4096, kick=8),
    "large": Config("large", 500, 27, 13, 11, 5, 120, "regional", 10, 20000, 10),
    "surge": Config("surge", 4000, 67, 33, 17, 8, 400, "disaster", 20, 1000, 10),
}
CONFIG_NUMBER = {"tiny": 1, "ontario": 2, "batched": 3, "large": 4, "surge": 5}


@dataclasses.dataclass
class Instance:
    """Plain arrays in the layout of `as_instance_desc` (include/airsched.h)."""
    travel_s: np.ndarray        # int32 [n_classes][n_locations][n_locations]
    class_is_heli: np.ndarray   # uint8 [n_classes]
    base_location: np.ndarray   # int32 [n_bases]
    vehicle_base: np.ndarray    # int32 [n_vehicles]
    vehicle_class: np.ndarray   # int32 [n_vehicles]
    pickup_loc: np.ndarray      # int32 [n_missions]
    delivery_loc: np.ndarray    # int32 [n_missions]
    deadline_s: np.ndarray      # int32 [n_missions]
    heli_only: np.ndarray       # uint8 [n_missions]
    flight_limit_s: int = FLIGHT_LIMIT_S
    day_length_s: int = DAY_S
    # planted feasible schedule (CSR: vehicle v owns route_missions[ptr[v]:ptr[v+1]])
    planted_ptr: np.ndarray | None = None
    planted_missions: np.ndarray | None = None
    seed: int = 0
    name: str = ""
    no_wait: int = 0            # f3 model variant: depart on arrival (reading #40)

    @property
    def n_missions(self) -> int:
        return int(self.pickup_loc.shape[0])

    @property
    def n_vehicles(self) -> int:
        return int(self.vehicle_base.shape[0])

    @property
    def n_locations(self) -> int:
        return int(self.travel_s.shape[1])

    @property
    def n_classes(self) -> int:
        return int(self.travel_s.shape[0])

    def vehicle_location(self) -> np.ndarray:
        return self.base_location[self.vehicle_base]


def haversine_km(lat1, lon1, lat2, lon2):
    """Eq. e1 numerator / 1 (§3): 2 r asin(sqrt(...)), degrees in."""
    p1, p2 = np.radians(lat1), np.radians(lat2)
    dphi = p2 - p1
    dlmb = np.radians(lon2) - np.radians(lon1)
    a = np.sin(dphi / 2.0) ** 2 + np.cos(p1) * np.cos(p2) * np.sin(dlmb / 2.0) ** 2
    return 2.0 * EARTH_RADIUS_KM * np.arcsin(np.sqrt(np.minimum(a, 1.0)))


def travel_matrix(lat: np.ndarray, lon: np.ndarray) -> np.ndarray:
    """Integer-second travel time per class: llround(km / speed * 3600) (reading #11)."""
    km = haversine_km(lat[:, None], lon[:, None], lat[None, :], lon[None, :])
    np.fill_diagonal(km, 0.0)
    out = np.empty((len(SPEED_KMH), len(lat), len(lat)), dtype=np.int32)
    for c, s in enumerate(SPEED_KMH):
        out[c] = np.floor(km / s * 3600.0 + 0.5).astype(np.int32)  # round half up (x >= 0)
    return out


def _region_points(rng: np.random.Generator, region: str, count: int):
    if region == "ontario":
        lat0, lat1, lon0, lon1 = _ONTARIO_BOX
        lat = np.empty(count)
        lon = np.empty(count)
        for i in range(count):
            u = rng.random()
            if u < 0.6:      # 60% around southern centres (survey §8(d))
                c = _ONTARIO_SOUTH[rng.integers(len(_ONTARIO_SOUTH))]
                lat[i] = c[0] + rng.normal(0, 0.35)
                lon[i] = c[1] + rng.normal(0, 0.5)
            elif u < 0.8:
                c = _ONTARIO_NORTH[rng.integers(len(_ONTARIO_NORTH))]
                lat[i] = c[0] + rng.normal(0, 0.35)
                lon[i] = c[1] + rng.normal(0, 0.5)
            else:
                lat[i] = rng.uniform(lat0, lat1)
                lon[i] = rng.uniform(lon0, lon1)
        return np.clip(lat, lat0, lat1), np.clip(lon, lon0, lon1)
    if region == "regional":     # ~300 x 300 km cluster around (44.5, -79.0)
        return rng.uniform(43.15, 45.85, count), rng.uniform(-80.9, -77.1, count)
    if region == "disaster":     # 60 km radius zone around (43.65, -79.38)
        r = 60.0 * np.sqrt(rng.random(count))
        th = rng.uniform(0, 2 * math.pi, count)
        return 43.65 + (r * np.sin(th)) / 111.0, -79.38 + (r * np.cos(th)) / (111.0 * math.cos(math.radians(43.65)))
    raise ValueError(region)


def generate(config: str | Config, seed: int | None = None, n_missions: int | None = None) -> Instance:
    """Generate one instance.  Retries deterministically (seed+1000*k) if planting fails."""
    cfg = CONFIGS[config] if isinstance(config, str) else config
    if n_missions is not None:
        cfg = dataclasses.replace(cfg, n_missions=n_missions)
    if seed is None:
        seed = SEED_BASE + CONFIG_NUMBER.get(cfg.name, 0)
    for k in range(64):
        inst = _try_generate(cfg, seed + 1000 * k)
        if inst is not None:
            return inst
    raise RuntimeError(f"could not plant a feasible instance for {cfg.name}")


def _try_generate(cfg: Config, seed: int) -> Instance | None:
    rng = np.random.default_rng(seed)
    F, B, n = cfg.n_facilities, cfg.n_bases, cfg.n_missions
    flat, flon = _region_points(rng, cfg.region, F)
    blat, blon = _region_points(rng, cfg.region, B)
    lat = np.concatenate([flat, blat])
    lon = np.concatenate([flon, blon])
    T = travel_matrix(lat, lon)
    NL = F + B
    base_location = np.arange(F, NL, dtype=np.int32)
    # bases 0..n_heli_bases-1 are helicopter bases, the rest plane bases
    base_class = np.array([0] * cfg.n_heli_bases + [1] * cfg.n_plane_bases, dtype=np.int32)
    heli_bases = np.flatnonzero(base_class == 0)
    plane_bases = np.flatnonzero(base_class == 1)
    vbase, vcls = [], []
    for i in range(cfg.n_heli_vehicles):
        vbase.append(heli_bases[i % len(heli_bases)]); vcls.append(0)
    for i in range(cfg.n_plane_vehicles):
        vbase.append(plane_bases[i % len(plane_bases)]); vcls.append(1)
    vehicle_base = np.array(vbase, dtype=np.int32)
    vehicle_class = np.array(vcls, dtype=np.int32)
    V = len(vbase)
    vloc = base_location[vehicle_base]

    K = max(2, min(cfg.locality, F))
    near_fac = np.argsort(T[0][:, :F], axis=1, kind="stable")  # facilities by distance from any location

    P = FLIGHT_LIMIT_S
    budget = int(0.9 * P)
    per_vehicle = max(1.0, n / V)
    slack_max = max(60, int(0.9 * DAY_S / per_vehicle))

    end_loc = vloc.copy()
    dep = np.zeros(V, dtype=np.int64)
    flight = np.zeros(V, dtype=np.int64)
    routes: list[list[int]] = [[] for _ in range(V)]
    pick = np.empty(n, np.int32)
    dele = np.empty(n, np.int32)
    w = np.empty(n, np.int32)
    heli = np.zeros(n, np.uint8)
    for j in range(n):
        placed = False
        for attempt in range(400):
            v = int(rng.integers(V))
            c = vcls[v]
            cand = near_fac[vloc[v]][:K]
            pk = int(cand[rng.integers(len(cand))])
            dcand = [x for x in near_fac[pk][:K + 1] if x != pk]
            dl = int(dcand[rng.integers(len(dcand))])
            leg = int(T[c][end_loc[v]][pk]) + int(T[c][pk][dl])
            ret = int(T[c][dl][vloc[v]])
            if flight[v] + leg + ret > budget:
                continue
            arrival = int(dep[v]) + leg
            slack = int(rng.integers(0, slack_max + 1)) if attempt < 300 else 0
            wj = max(1, arrival + slack)
            if wj + ret > DAY_S:
                wj = max(1, arrival)
                if wj + ret > DAY_S:
                    continue
            pick[j], dele[j], w[j] = pk, dl, wj
            if c == 0 and rng.random() < 0.25:   # heli_only ~ Bernoulli(0.25) on heli routes
                heli[j] = 1
            routes[v].append(j)
            end_loc[v] = dl
            dep[v] = wj
            flight[v] += leg
            placed = True
            break
        if not placed:
            return None
    # shuffle mission ids
    perm = rng.permutation(n)          # new id of old mission j is perm[j]
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n)
    pick, dele, w, heli = pick[inv], dele[inv], w[inv], heli[inv]
    ptr = [0]
    ms: list[int] = []
    for v in range(V):
        ms.extend(int(perm[j]) for j in routes[v])
        ptr.append(len(ms))
    return Instance(
        travel_s=T, class_is_heli=np.array(CLASS_IS_HELI, np.uint8),
        base_location=base_location, vehicle_base=vehicle_base, vehicle_class=vehicle_class,
        pickup_loc=pick.astype(np.int32), delivery_loc=dele.astype(np.int32),
        deadline_s=w.astype(np.int32), heli_only=heli.astype(np.uint8),
        planted_ptr=np.array(ptr, np.int32), planted_missions=np.array(ms, np.int32),
        seed=seed, name=cfg.name)


def splitmix64_seeds(count: int, base: int = 1) -> np.ndarray:
    """Run seeds 1..count; plain integers, no generator arithmetic."""
    return np.arange(base, base + count, dtype=np.uint64)
