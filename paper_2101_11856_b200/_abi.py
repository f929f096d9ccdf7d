"""ctypes declarations of include/lbmg.h (shared by the product binding and
by the oracle adapter loader in tests, which reuses the scene struct)."""
from __future__ import annotations

import ctypes as C


class Face(C.Structure):
    _fields_ = [("condition", C.c_int), ("velocity", C.c_double * 3)]


class Mesh(C.Structure):
    _fields_ = [
        ("type", C.c_int),
        ("center", C.c_double * 3), ("lo", C.c_double * 3), ("hi", C.c_double * 3), ("origin", C.c_double * 3),
        ("radius", C.c_double), ("subdivisions", C.c_int), ("fins", C.c_int),
        ("fin_length", C.c_double), ("fin_height", C.c_double), ("fin_spacing", C.c_double),
        ("size", C.c_double), ("plane_z", C.c_double),
    ]


class SolidConfigC(C.Structure):
    _fields_ = [
        ("mesh", Mesh), ("poisson_radius", C.c_double), ("sampling", C.c_int), ("has_motion", C.c_int),
        ("linear_velocity", C.c_double * 3), ("angular_velocity", C.c_double * 3), ("center", C.c_double * 3),
    ]


class SceneConfigC(C.Structure):
    _fields_ = [
        ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
        ("viscosity", C.c_double), ("kind", C.c_int), ("high_order_rate", C.c_double),
        ("policy", C.c_int), ("policy_eps0", C.c_double),
        ("has_explicit_rates", C.c_int), ("rates", C.c_double * 27),
        ("faces", Face * 6), ("body_force", C.c_double * 3),
        ("n_solids", C.c_int), ("solids", C.POINTER(SolidConfigC)),
        ("init", C.c_int), ("init_density", C.c_double), ("init_velocity", C.c_double * 3),
        ("tg_u_max", C.c_double), ("regions", C.c_int), ("threads_per_region", C.c_uint),
        ("alpha", C.c_size_t), ("block_edge", C.c_int), ("ib_mode", C.c_int), ("seed", C.c_uint64),
    ]


class EmitterC(C.Structure):  # lbmg_emitter (TracerEmitter, tracer.hpp:14-17)
    _fields_ = [("lo", C.c_double * 3), ("hi", C.c_double * 3), ("rate", C.c_int)]


class StatusC(C.Structure):
    _fields_ = [("ok", C.c_int), ("mach_warning", C.c_int), ("step", C.c_long), ("reason", C.c_char * 120)]


class TimingRowC(C.Structure):
    _fields_ = [("phase", C.c_char * 24), ("step", C.c_long), ("seconds", C.c_double)]


# enum values (lbmg.h)
BGK, RAW_MRT, CENTRAL_MRT = 0, 1, 2
POLICY_CONSTANT, POLICY_RELAX_TOWARD_ONE = 0, 1
NOSLIP, INLET, OUTFLOW, PERIODIC = 0, 1, 2, 3
MESH_SPHERE, MESH_BOX, MESH_FIN_COMB, MESH_QUAD = 0, 1, 2, 3
SAMPLING_DART, SAMPLING_ELIMINATION = 0, 1
INIT_UNIFORM, INIT_TAYLOR_GREEN = 0, 1
IB_ATOMIC, IB_DETERMINISTIC = 0, 1
PHASE_PRE, PHASE_MID, PHASE_FLUID_EDGE, PHASE_FLUID_BULK, PHASE_END = range(5)

ERR = {1: "ConfigError", 2: "CudaError", 3: "OutOfMemory", 4: "IoError", 5: "StateError"}
