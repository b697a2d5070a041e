"""Python mirror of the reference's ``moseslab`` hot-path API over the C ABI.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/moseslab/{model,lottery,search}.hpp; every call
goes through ``libmoses_gpu.so`` (include/moses_gpu.h). There is no CPU
fallback: importing this module on a machine without the built library or a
B200 raises.

Value model: ``CostModelParams`` is the host value (dims + flat float64 params
+ momentum, the reference flat order). ``DeviceModel`` is a device handle; the
free functions accept either and upload on demand, so reference-style code
(`predict(params, features)`) works unchanged, while hot loops keep a
``DeviceModel`` resident.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmoses_gpu.so")

# moseslab::ErrorCode names (errors.hpp:10-36), indexed by ordinal
ERROR_NAMES = [
    "invalid-task", "invalid-config", "space-too-large", "immutable-space", "bad-dims",
    "dim-mismatch", "shape-mismatch", "version-mismatch", "corrupt-stream", "empty-dataset",
    "invalid-ratio", "unnormalized-threshold", "adversary-disabled", "unstable-decay",
    "infeasible-split", "zero-mean", "insufficient-batches", "budget-infeasible",
    "missing-reference-strategy", "mismatched-runs", "empty-rows", "parse-error",
    "missing-field", "io-error", "usage-error",
]
LIB_ERRORS = {100: "cuda-error", 101: "no-device", 102: "capacity", 103: "invalid-argument"}

PREC_BF16, PREC_TF32, PREC_FP32, PREC_BF16X3 = 0, 1, 2, 3  # FP32: 3xTF32, BF16X3: split bf16 operands
THRESHOLD, RATIO = 1, 2
DTYPE_F32, DTYPE_BF16, DTYPE_F64 = 0, 1, 2


def input_dtype(precision: int) -> int:
    """Element type of device-resident input rows for a handle of this precision (moses_gpu.h)."""
    return DTYPE_BF16 if precision == PREC_BF16 else DTYPE_F32


class MosesError(RuntimeError):
    """moseslab::Error equivalent: .code is the reference's error_code_name."""

    def __init__(self, status: int, message: str):
        if 1 <= status <= len(ERROR_NAMES):
            self.code = ERROR_NAMES[status - 1]
        else:
            self.code = LIB_ERRORS.get(status, f"status-{status}")
        self.status = status
        super().__init__(f"{self.code}: {message}")


_lib = None


def lib():
    """Load the CUDA library. Fails loudly if it is missing (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing; run `python -m paper_2201_05752_b200.build`")
    L = C.CDLL(_LIB_PATH)
    vp, i32, i64, u64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
    sig = {
        "moses_last_error": (C.c_char_p, []),
        "moses_version": (C.c_char_p, []),
        "moses_kernel_launches": (i64, []),
        "moses_device_check": (C.c_int, []),
        "moses_param_count": (i64, [vp, i32]),
        "moses_init_random": (C.c_int, [vp, i32, u64, i32, vp]),
        "moses_model_create": (C.c_int, [vp, i32, i32, i64, vp]),
        "moses_model_destroy": (C.c_int, [vp]),
        "moses_model_upload": (C.c_int, [vp, vp, vp, i64]),
        "moses_model_download": (C.c_int, [vp, vp, vp, i64]),
        "moses_model_copy": (C.c_int, [vp, vp]),
        "moses_model_synchronize": (C.c_int, [vp]),
        "moses_packed_ld": (i64, [vp]),
        "moses_predict": (C.c_int, [vp, vp, i64, i32, vp]),
        "moses_penultimate": (C.c_int, [vp, vp, i64, i32, vp]),
        "moses_predict_device": (C.c_int, [vp, vp, i32, i64, i64, vp]),
        "moses_predict_pooled": (C.c_int, [vp, vp, i64, i32, vp, i64, vp]),
        "moses_gradients": (C.c_int, [vp, vp, vp, i64, i32, vp, dbl, vp]),
        "moses_gradients_device": (C.c_int, [vp, vp, i64, vp, i64, vp]),
        "moses_set_async": (C.c_int, [i32]),
        "moses_train_graph_create": (C.c_int, [vp, vp, i64, vp, i64, i64, dbl, dbl, i32]),
        "moses_train_graph_launch": (C.c_int, [vp, i64]),
        "moses_train_graph_create_pooled": (C.c_int, [vp, vp, i64, vp, vp, i64, i64, i64, dbl, dbl, i32]),
        "moses_gradients_pooled": (C.c_int, [vp, vp, i64, i32, vp, i64, vp, vp]),
        "moses_synth_offsets": (C.c_int, [u64, i64, i32, vp]),
        "moses_train_graph_kernels": (C.c_int, []),
        "moses_profile_begin": (C.c_int, []),
        "moses_profile_end": (C.c_int, [vp, vp, i32]),
        "moses_gradients_download": (C.c_int, [vp, vp, i64]),
        "moses_gradients_upload": (C.c_int, [vp, vp, i64]),
        "moses_objective": (C.c_int, [vp, vp, vp, i64, i32, vp, dbl, vp]),
        "moses_apply_update": (C.c_int, [vp, dbl, dbl, vp, i64, i32]),
        "moses_train_step": (C.c_int, [vp, vp, vp, i64, i32, dbl, dbl, vp]),
        "moses_train_step_device": (C.c_int, [vp, vp, i64, vp, i64, dbl, dbl, vp]),
        "moses_ranking_accuracy": (C.c_int, [vp, vp, vp, vp, i32, i32, vp, vp, vp]),
        "moses_ranking_loss": (C.c_int, [vp, vp, i64, vp, vp]),
        "moses_adam_update": (C.c_int, [vp, dbl, dbl, dbl, dbl, i32, vp, i64]),
        "moses_xi_scores": (C.c_int, [vp, i32, vp, i64]),
        "moses_partition": (C.c_int, [vp, i32, dbl, i32, vp, i64, vp]),
        "moses_xi_upload": (C.c_int, [vp, vp, i64, i32]),
        "moses_mask_upload": (C.c_int, [vp, vp, i64]),
        "moses_transferable_step": (C.c_int, [vp, dbl]),
        "moses_variant_decay": (C.c_int, [vp, dbl, dbl]),
        "moses_lottery_step": (C.c_int, [vp, i32, dbl, i32, dbl, dbl, vp, i64, vp]),
        "moses_adversary_create": (C.c_int, [vp, i64, i32, i32, dbl, vp]),
        "moses_adversary_destroy": (C.c_int, [vp]),
        "moses_adversary_get": (C.c_int, [vp, vp, i32, vp]),
        "moses_adversary_set": (C.c_int, [vp, vp, i32, dbl]),
        "moses_adversarial_term": (C.c_int, [vp, vp, i64, vp, i64, i32, dbl, vp, vp]),
        "moses_adversarial_step": (C.c_int, [vp, vp, vp, i64, i32, dbl, vp, vp]),
        "moses_discriminator_cross_entropy": (C.c_int, [vp, i64, vp, i64, vp]),
        "moses_topk": (C.c_int, [vp, i64, i64, vp]),
        "moses_topk_device": (C.c_int, [vp, i64, i64, vp]),
        "moses_select_batch": (i64, [vp, i64, vp, i64, i64, vp]),
        "moses_segment_sum": (C.c_int, [vp, i64, i32, vp, i64, vp]),
        "moses_segment_sum_device": (C.c_int, [vp, i32, i64, i32, vp, i64, vp]),
        "moses_mmd2": (C.c_int, [vp, i64, vp, i64, i32, dbl, vp]),
        "moses_mmd2_device": (C.c_int, [vp, i64, vp, i64, i32, i64, dbl, vp]),
        "moses_gradients_mmd": (C.c_int, [vp, vp, vp, i64, i32, vp, i64, dbl, dbl, vp]),
        "moses_mmd2_grad": (C.c_int, [vp, i64, vp, i64, i32, dbl, vp, vp, vp]),
        "moses_encode_configs_device": (C.c_int, [vp, vp, vp, vp, i32, C.c_uint64, i64, i32, vp, i64, i32, vp, vp]),
        "moses_measure_configs_device": (C.c_int, [vp, i32, C.c_char_p, C.c_char_p, vp, vp, vp, vp, i32, C.c_uint64,
                                                   C.c_uint64, i64, vp, vp, vp, vp, vp]),
        "moses_true_best": (C.c_int, [vp, vp, vp, vp, vp, i32, vp, vp]),
        "moses_train_step_pooled_async": (C.c_int, [vp, vp, i64, i32, vp, i64, vp, dbl, dbl, vp]),
        "moses_encode_configs": (C.c_int, [vp, vp, vp, vp, i32, C.c_uint64, i64, vp, vp]),
        "moses_lottery_step_adam": (C.c_int, [vp, i32, dbl, i32, dbl, dbl, dbl, dbl, i32, dbl, vp, i64, vp]),
        "moses_generate_dataset_device": (C.c_int, [vp, i32, C.c_char_p, C.c_char_p, vp, vp, vp, vp, i32, i64, u64,
                                                    i32, vp, i64, i32, vp, vp, vp, vp, vp]),
        "moses_encode_values_device": (C.c_int, [vp, vp, vp, vp, i32, vp, i64, i32, vp, i64, i32, vp, vp]),
        "moses_epoch_seed": (u64, [u64, u64]),
        "moses_ranking_plan": (C.c_int, [vp, i64, vp, i32, i32, u64, vp, vp, vp, vp, vp]),
        "moses_replay_rows": (C.c_int, [i64, i64, u64, vp, vp]),
        "moses_train_plan_device": (C.c_int, [vp, vp, i64, vp, i64, vp, vp, i64, dbl, dbl, vp]),
        "moses_pretrain_device": (C.c_int, [vp, vp, i64, vp, vp, i64, vp, i32, i32, u64, i32, dbl, dbl, vp, vp]),
        "moses_pretrain_jobs": (C.c_int, [i32, vp, vp, vp, i64, vp, vp, i64, vp, i32, i32, i32, dbl, dbl, i32, vp, vp]),
        "moses_pretrain_jobs_mapped": (C.c_int, [i32, vp, vp, vp, i64, vp, vp, i64, vp, i32, i32, i32, dbl, dbl, i32,
                                                 vp, vp]),
        "moses_pretrain": (C.c_int, [vp, i32, vp, vp, vp, vp, vp, i32, vp, vp, vp, i64, i32, u64, i32, dbl, dbl, vp, vp]),
        "moses_moses_step": (C.c_int, [vp, vp, vp, vp, i64, i32, dbl, i32, dbl, i32, dbl, dbl, vp, vp, vp]),
        "moses_evolve": (C.c_int, [vp, vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, dbl, u64, vp, vp, i64, vp]),
        "moses_tune_task": (C.c_int, [vp, i32, vp, vp, vp, u64, vp, i64, vp]),
        "moses_tune_jobs": (C.c_int, [i32, vp, vp, vp, vp, vp, i32, vp, vp, vp, i64, i32, vp]),
        "moses_records_create": (C.c_int, [vp]),
        "moses_records_read": (C.c_int, [C.c_char_p, vp]),
        "moses_records_destroy": (None, [vp]),
        "moses_records_append": (C.c_int, [vp, C.c_char_p, C.c_char_p, i64, i32, vp, vp, vp, vp, vp]),
        "moses_records_write": (C.c_int, [vp, C.c_char_p]),
        "moses_records_shape": (C.c_int, [vp, vp, vp, vp, vp]),
        "moses_records_task_id": (C.c_char_p, [vp, i32]),
        "moses_records_device_id": (C.c_char_p, [vp, i32]),
        "moses_records_export": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "moses_debug_force_serial_sampling": (C.c_int, [i32]),
        "moses_synth_features_device": (C.c_int, [u64, i64, i64, i32, i32, vp, i64]),
        "moses_synth_labels_device": (C.c_int, [u64, i64, i64, vp]),
        "moses_serialize": (i64, [vp, i32, vp, vp, vp, i64]),
        "moses_deserialize": (C.c_int, [vp, i64, vp, vp, vp, i64]),
        "moses_write_mask": (i64, [vp, i64, i32, i32, dbl, vp, i64]),
        "moses_read_mask": (C.c_int, [vp, i64, vp, i64, vp, vp, vp, vp]),
        "moses_model_device_ptrs": (C.c_int, [vp, vp, vp, vp]),
        "moses_model_stream": (C.c_int, [vp, vp]),
        "moses_comm_unique_id": (C.c_int, [vp, i64]),
        "moses_comm_init_rank": (C.c_int, [vp, i32, i32, vp]),
        "moses_comm_init_all": (C.c_int, [i32, vp, vp]),
        "moses_comm_destroy": (C.c_int, [vp]),
        "moses_comm_info": (C.c_int, [vp, vp, vp, vp]),
        "moses_model_set_comm": (C.c_int, [vp, vp, i32]),
        "moses_dp_allreduce_gradients": (C.c_int, [vp, i32]),
        "moses_dp_train_step": (C.c_int, [vp, vp, i64, vp, i64, dbl, dbl, vp]),
        "moses_dp_exact_forward": (C.c_int, [vp, vp, i64, vp, i64, vp, vp]),
        "moses_dp_exact_rank": (C.c_int, [vp, vp, vp, i64, i64, vp]),
        "moses_dp_exact_backward": (C.c_int, [vp, i64, vp, vp]),
        "moses_topk_sharded": (C.c_int, [vp, vp, i64, i64, i64, vp]),
        "moses_debug_gemm": (C.c_int, [C.c_int] * 4 + [vp, C.c_longlong, C.c_int, vp, C.c_longlong, C.c_int, C.c_int,
                                                       vp, C.c_longlong, vp, C.c_int, C.c_int, vp, C.c_longlong]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def exported_symbols() -> list[str]:
    return [n for n in lib().__dict__ if n.startswith("moses_")]


def _ck(rc: int):
    if rc != 0:
        raise MosesError(rc, lib().moses_last_error().decode(errors="replace"))


def _p(a):
    return None if a is None else a.ctypes.data


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _dims(dims):
    return np.ascontiguousarray(dims, dtype=np.int32)


def kernel_launches() -> int:
    return lib().moses_kernel_launches()


PROFILE_CATS = ["gemm_fwd", "gemm_dgrad", "gemm_wgrad", "rank", "head", "update", "select", "topk", "other"]


def profile_begin():
    _ck(lib().moses_profile_begin())


def profile_end() -> dict:
    ms = np.zeros(len(PROFILE_CATS))
    cnt = np.zeros(len(PROFILE_CATS), dtype=np.int64)
    _ck(lib().moses_profile_end(_p(ms), _p(cnt), len(PROFILE_CATS)))
    return {c: (float(ms[i]), int(cnt[i])) for i, c in enumerate(PROFILE_CATS)}


# ---------------------------------------------------------------- values (model.hpp:19-48)
@dataclass
class CostModelParams:
    dims: list
    params: np.ndarray                # flat, reference order
    momentum: Optional[np.ndarray] = None

    def __post_init__(self):
        self.params = _f64(self.params)
        if self.momentum is None:
            self.momentum = np.zeros_like(self.params)
        self.momentum = _f64(self.momentum)

    def copy(self):
        return CostModelParams(list(self.dims), self.params.copy(), self.momentum.copy())

    # views per level, reference shapes: w[l] is dims[l+1] x dims[l] (column-major storage)
    def level_offset(self, l):
        return int(sum(self.dims[k] * self.dims[k + 1] + self.dims[k + 1] for k in range(l)))

    def w(self, l):
        o, fi, fo = self.level_offset(l), self.dims[l], self.dims[l + 1]
        return self.params[o:o + fi * fo].reshape(fi, fo).T

    def b(self, l):
        o, fi, fo = self.level_offset(l), self.dims[l], self.dims[l + 1]
        return self.params[o + fi * fo:o + fi * fo + fo]


@dataclass
class TrainHyper:  # model.hpp:27-35
    learning_rate: float = 0.001
    weight_decay: float = 0.01
    max_epochs: int = 30
    batch_size: int = 512
    momentum: float = 0.9
    adversary_beta: float = 0.01
    seed: int = 0


@dataclass
class RankingBatch:  # model.hpp:39-43
    features: np.ndarray
    labels: np.ndarray
    task_id: str = ""


@dataclass
class XiScores:  # lottery.hpp:15-18
    xi: np.ndarray
    normalized: bool = False


@dataclass
class ParamMask:  # lottery.hpp:25-32
    transferable: np.ndarray
    phase: int = 0
    mode: int = RATIO
    value: float = 0.0

    def popcount(self) -> int:
        return int(np.count_nonzero(self.transferable))


def param_count(dims) -> int:
    d = _dims(dims)
    n = lib().moses_param_count(_p(d), len(d))
    if n < 0:
        _ck(int(-n))
    return int(n)


def init_random(dims, seed: int, strict: bool = True) -> CostModelParams:
    """model.cpp:147-167 (bit-exact keyed SplitMix64 draw order)."""
    d = _dims(dims)
    n = param_count(dims) if len(dims) >= 3 else 0
    out = np.zeros(max(n, 1), dtype=np.float64)
    _ck(lib().moses_init_random(_p(d), len(d), seed, int(strict), _p(out)))
    return CostModelParams(list(dims), out[:n])


# ---------------------------------------------------------------- device handles
class DeviceModel:
    """Device-resident cost model (one CUDA stream + workspaces per handle)."""

    def __init__(self, params: CostModelParams, precision: int = PREC_TF32, max_rows: int = 4096):
        self.dims = list(params.dims)
        d = _dims(self.dims)
        h = C.c_void_p()
        _ck(lib().moses_model_create(_p(d), len(d), precision, max_rows, C.byref(h)))
        self.h = h
        self.precision = precision
        self.P = param_count(self.dims)
        self.upload(params)

    def upload(self, params: CostModelParams):
        _ck(lib().moses_model_upload(self.h, _p(params.params), _p(params.momentum), self.P))

    def download(self) -> CostModelParams:
        w = np.zeros(self.P)
        m = np.zeros(self.P)
        _ck(lib().moses_model_download(self.h, _p(w), _p(m), self.P))
        return CostModelParams(list(self.dims), w, m)

    def gradients(self) -> np.ndarray:
        g = np.zeros(self.P)
        _ck(lib().moses_gradients_download(self.h, _p(g), self.P))
        return g

    def set_gradients(self, g):
        g = _f64(g)
        _ck(lib().moses_gradients_upload(self.h, _p(g), self.P))

    @property
    def packed_ld(self) -> int:
        return int(lib().moses_packed_ld(self.h))

    def close(self):
        if getattr(self, "h", None):
            lib().moses_model_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _as_device(model, precision=PREC_TF32, rows=4096):
    if isinstance(model, DeviceModel):
        return model, False
    return DeviceModel(model, precision, max(rows, 1)), True


class AdversaryState:
    """lottery.hpp:36-42 — logistic discriminator + frozen replay rows (device)."""

    def __init__(self, replay_features, penultimate_dim: int, seed: int = 0, step_size: float = 0.1):
        r = _f64(replay_features)
        if r.ndim != 2:
            r = r.reshape(0, 0) if r.size == 0 else r
        h = C.c_void_p()
        _ck(lib().moses_adversary_create(_p(r), r.shape[0], r.shape[1] if r.ndim == 2 else 0, penultimate_dim,
                                         step_size, C.byref(h)))
        self.h = h
        self.width = penultimate_dim
        self.replay_features = r
        self.step_size = step_size
        self.seed = seed

    @property
    def weight(self):
        w = np.zeros(self.width)
        b = C.c_double()
        _ck(lib().moses_adversary_get(self.h, _p(w), self.width, C.byref(b)))
        return w

    @property
    def bias(self):
        w = np.zeros(self.width)
        b = C.c_double()
        _ck(lib().moses_adversary_get(self.h, _p(w), self.width, C.byref(b)))
        return b.value

    def set(self, weight, bias):
        w = _f64(weight)
        _ck(lib().moses_adversary_set(self.h, _p(w), self.width, float(bias)))

    def __del__(self):
        try:
            if self.h:
                lib().moses_adversary_destroy(self.h)
        except Exception:
            pass


def make_adversary(replay_features, penultimate_dim, seed=0, step_size=0.1) -> AdversaryState:
    """lottery.cpp:166-180"""
    return AdversaryState(replay_features, penultimate_dim, seed, step_size)


# ---------------------------------------------------------------- model.hpp functions
def predict(model, features) -> np.ndarray:
    """model.cpp:169-175"""
    x = _f64(features)
    n, D = x.shape
    dm, tmp = _as_device(model, rows=n)
    out = np.zeros(n)
    try:
        _ck(lib().moses_predict(dm.h, _p(x), n, D, _p(out)))
    finally:
        if tmp:
            dm.close()
    return out


def penultimate_activations(model, features) -> np.ndarray:
    """model.cpp:177-183"""
    x = _f64(features)
    n, D = x.shape
    dm, tmp = _as_device(model, rows=n)
    out = np.zeros((n, dm.dims[-2]))
    try:
        _ck(lib().moses_penultimate(dm.h, _p(x), n, D, _p(out)))
    finally:
        if tmp:
            dm.close()
    return out


def predict_pooled(model, stmt_features, offsets) -> np.ndarray:
    x = _f64(stmt_features)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    dm, tmp = _as_device(model, rows=x.shape[0])
    out = np.zeros(len(off) - 1)
    try:
        _ck(lib().moses_predict_pooled(dm.h, _p(x), x.shape[0], x.shape[1], _p(off), len(off) - 1, _p(out)))
    finally:
        if tmp:
            dm.close()
    return out


def pairwise_ranking_loss(scores, labels) -> float:
    """model.cpp:185-190"""
    s, y = _f64(scores), _f64(labels)
    if s.shape != y.shape:
        raise MosesError(6, "scores/labels length mismatch")
    loss = C.c_double()
    pairs = C.c_int64()
    _ck(lib().moses_ranking_loss(_p(s), _p(y), len(s), C.byref(loss), C.byref(pairs)))
    return loss.value


def gradients(model, batch: RankingBatch, adversary: Optional[AdversaryState] = None, beta: float = 0.0,
              want_loss: bool = False):
    """model.cpp:192-244. Returns the flat gradient (and the loss when want_loss)."""
    x, y = _f64(batch.features), _f64(batch.labels)
    n = x.shape[0]
    D = x.shape[1] if x.ndim == 2 else 0
    if y.shape[0] != n:
        raise MosesError(6, "batch rows != label count")
    rows = n + (adversary.replay_features.shape[0] if adversary is not None else 0)
    dm, tmp = _as_device(model, rows=rows)
    loss = C.c_double()
    try:
        _ck(lib().moses_gradients(dm.h, _p(x), _p(y), n, D, adversary.h if adversary else None, beta,
                                  C.byref(loss)))
        g = dm.gradients()
    finally:
        if tmp:
            dm.close()
    return (g, loss.value) if want_loss else g


def gradients_pooled(model, stmt_features, offsets, labels, want_loss=False):
    """Pooled (TenSet-shaped) gradient: statement rows, CSR program offsets, one label per program."""
    x, y = _f64(stmt_features), _f64(labels)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    dm, tmp = _as_device(model, rows=max(x.shape[0], 1))
    loss = C.c_double()
    try:
        _ck(lib().moses_gradients_pooled(dm.h, _p(x), x.shape[0], x.shape[1], _p(off), len(off) - 1, _p(y),
                                         C.byref(loss)))
        g = dm.gradients()
    finally:
        if tmp:
            dm.close()
    return (g, loss.value) if want_loss else g


def synth_offsets(seed, programs, max_stmts=8) -> np.ndarray:
    out = np.zeros(programs + 1, dtype=np.int64)
    _ck(lib().moses_synth_offsets(seed, programs, max_stmts, _p(out)))
    return out


def objective(model, batch: RankingBatch, adversary=None, beta=0.0) -> float:
    """model.cpp:246-261"""
    x, y = _f64(batch.features), _f64(batch.labels)
    rows = x.shape[0] + (adversary.replay_features.shape[0] if adversary is not None else 0)
    dm, tmp = _as_device(model, rows=rows)
    out = C.c_double()
    try:
        _ck(lib().moses_objective(dm.h, _p(x), _p(y), x.shape[0], x.shape[1], adversary.h if adversary else None,
                                  beta, C.byref(out)))
    finally:
        if tmp:
            dm.close()
    return out.value


def apply_update(model: DeviceModel, hyper: TrainHyper = TrainHyper(), mask: Optional[ParamMask] = None,
                 use_momentum: bool = False, grads=None):
    """model.cpp:263-296 on the handle (uses its device gradients unless `grads` is given)."""
    if grads is not None:
        model.set_gradients(grads)
    m = None if mask is None else np.ascontiguousarray(mask.transferable, dtype=np.uint8)
    _ck(lib().moses_apply_update(model.h, hyper.learning_rate, hyper.momentum, _p(m), 0 if m is None else len(m),
                                 int(use_momentum)))


def ranking_accuracy(model, batches: Sequence[RankingBatch]) -> float:
    """model.cpp:298-312"""
    if not batches:
        return 0.0
    x = np.concatenate([_f64(b.features) for b in batches])
    y = np.concatenate([_f64(b.labels) for b in batches])
    off = np.zeros(len(batches) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(b.labels) for b in batches])
    dm, tmp = _as_device(model, rows=4096)
    acc = C.c_double()
    pairs = C.c_int64()
    conc = C.c_int64()
    try:
        _ck(lib().moses_ranking_accuracy(dm.h, _p(x), _p(y), _p(off), len(batches), x.shape[1], C.byref(acc),
                                         C.byref(pairs), C.byref(conc)))
    finally:
        if tmp:
            dm.close()
    return acc.value


# ---------------------------------------------------------------- lottery.hpp functions
def xi_scores(model: DeviceModel, normalize: bool, grads=None) -> XiScores:
    """lottery.cpp:35-57 (with the handle's params and device gradients)."""
    if grads is not None:
        model.set_gradients(grads)
    out = np.zeros(model.P)
    _ck(lib().moses_xi_scores(model.h, int(normalize), _p(out), model.P))
    return XiScores(out, normalize)


def partition(model: DeviceModel, xi: Optional[XiScores], mode: int, value: float, phase: int) -> ParamMask:
    """lottery.cpp:59-90. If `xi` is given it is uploaded (identical-input parity path)."""
    if xi is not None:
        x = _f64(xi.xi)
        if len(x) == 0:
            raise MosesError(7, "empty score array")
        _ck(lib().moses_xi_upload(model.h, _p(x), len(x), int(xi.normalized)))
    out = np.zeros(model.P, dtype=np.uint8)
    pop = C.c_int64()
    _ck(lib().moses_partition(model.h, mode, value, phase, _p(out), model.P, C.byref(pop)))
    return ParamMask(out.astype(bool), phase, mode, value)


def transferable_step(model: DeviceModel, mask: Optional[ParamMask], alpha: float, grads=None):
    """lottery.cpp:92-97"""
    if grads is not None:
        model.set_gradients(grads)
    if mask is not None:
        m = np.ascontiguousarray(mask.transferable, dtype=np.uint8)
        _ck(lib().moses_mask_upload(model.h, _p(m), len(m)))
    _ck(lib().moses_transferable_step(model.h, alpha))


def variant_decay(model: DeviceModel, mask: Optional[ParamMask], alpha: float, lam: float):
    """lottery.cpp:99-120"""
    if mask is not None:
        m = np.ascontiguousarray(mask.transferable, dtype=np.uint8)
        _ck(lib().moses_mask_upload(model.h, _p(m), len(m)))
    _ck(lib().moses_variant_decay(model.h, alpha, lam))


def lottery_step_adam(model, mode: int, value: float, phase: int, lr: float, b1: float, b2: float, eps: float,
                      step: int, lam: float) -> "ParamMask":
    """lottery_step with masked Adam on the transferable scalars (decay 1 - lr*lam on the rest)."""
    out = np.zeros(model.P, dtype=np.uint8)
    pop = C.c_int64()
    _ck(lib().moses_lottery_step_adam(model.h, mode, value, phase, lr, b1, b2, eps, step, lam, _p(out), model.P,
                                      C.byref(pop)))
    return ParamMask(out.astype(bool), phase, mode, value)


def lottery_step(model: DeviceModel, mode: int, value: float, phase: int, alpha: float, lam: float) -> ParamMask:
    """tuner.cpp:258-262 fused: xi -> partition -> transferable_step -> variant_decay."""
    out = np.zeros(model.P, dtype=np.uint8)
    pop = C.c_int64()
    _ck(lib().moses_lottery_step(model.h, mode, value, phase, alpha, lam, _p(out), model.P, C.byref(pop)))
    return ParamMask(out.astype(bool), phase, mode, value)


def discriminator_cross_entropy(z_source, z_target) -> float:
    """lottery.cpp:207-218"""
    zs, zt = _f64(z_source), _f64(z_target)
    out = C.c_double()
    _ck(lib().moses_discriminator_cross_entropy(_p(zs), len(zs), _p(zt), len(zt), C.byref(out)))
    return out.value


@dataclass
class AdversarialResult:
    discriminator_loss: float = 0.0
    confusion_contribution: float = 0.0


def adversarial_term(adversary: AdversaryState, hidden_source, hidden_target, beta: float) -> AdversarialResult:
    """lottery.cpp:135-164"""
    hs, ht = _f64(hidden_source), _f64(hidden_target)
    ms = hs.shape[0] if hs.ndim == 2 else 0
    nt = ht.shape[0] if ht.ndim == 2 else 0
    width = hs.shape[1] if hs.ndim == 2 and ms else (ht.shape[1] if ht.ndim == 2 and nt else adversary.width)
    if ht.ndim == 2 and nt and ht.shape[1] != width:
        raise MosesError(6, "activation width != discriminator width")
    dl, cf = C.c_double(), C.c_double()
    _ck(lib().moses_adversarial_term(adversary.h, _p(hs), ms, _p(ht), nt, width, beta, C.byref(dl), C.byref(cf)))
    return AdversarialResult(dl.value, cf.value)


def adversarial_step(adversary: AdversaryState, model: DeviceModel, target_features, beta: float):
    """tuner.cpp:252-256: penultimate activations of replay + target under the current params, then the step."""
    x = _f64(target_features)
    dl, cf = C.c_double(), C.c_double()
    _ck(lib().moses_adversarial_step(adversary.h, model.h, _p(x), x.shape[0], x.shape[1], beta, C.byref(dl),
                                     C.byref(cf)))
    return AdversarialResult(dl.value, cf.value)


# ---------------------------------------------------------------- search.hpp
def topk(scores, k: int) -> np.ndarray:
    """(score desc, index asc) order of search.cpp:32-37 over a candidate pool."""
    s = _f64(scores)
    k = min(int(k), len(s))
    out = np.zeros(max(k, 1), dtype=np.int64)
    _ck(lib().moses_topk(_p(s), len(s), k, _p(out)))
    return out[:k]


def select_batch(ordered_hashes, already_measured, batch_size: int) -> np.ndarray:
    """search.cpp:82-95 over a score-ordered list of config hashes: returns positions kept."""
    h = np.ascontiguousarray(ordered_hashes, dtype=np.uint64)
    m = np.ascontiguousarray(sorted(already_measured), dtype=np.uint64)
    out = np.zeros(max(int(batch_size), 1), dtype=np.int64)
    n = lib().moses_select_batch(_p(h), len(h), _p(m) if len(m) else None, len(m), batch_size, _p(out))
    if n < 0:
        _ck(int(-n))
    return out[:n]


# ---------------------------------------------------------------- extensions
def segment_sum(h, offsets) -> np.ndarray:
    h = _f64(h)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    out = np.zeros((len(off) - 1, h.shape[1]))
    _ck(lib().moses_segment_sum(_p(h), h.shape[0], h.shape[1], _p(off), len(off) - 1, _p(out)))
    return out


def mmd2(xs, xt, sigma: float) -> float:
    xs, xt = _f64(xs), _f64(xt)
    out = C.c_double()
    _ck(lib().moses_mmd2(_p(xs), xs.shape[0], _p(xt), xt.shape[0], xs.shape[1], sigma, C.byref(out)))
    return out.value


def mmd2_grad(xs, xt, sigma: float):
    """MMD^2 and its gradient w.r.t. every source / target row (moses_mmd2_grad)."""
    xs, xt = _f64(xs), _f64(xt)
    val = C.c_double()
    gs = np.zeros_like(xs)
    gt = np.zeros_like(xt)
    _ck(lib().moses_mmd2_grad(_p(xs), xs.shape[0], _p(xt), xt.shape[0], xs.shape[1], sigma, C.byref(val), _p(gs),
                              _p(gt)))
    return val.value, gs, gt


def gradients_mmd(model, batch: RankingBatch, source_features, beta: float, sigma: float, want_loss=False):
    """gradients() with beta * MMD^2(H_source, H_batch) as the domain term (moses_gradients_mmd)."""
    x, y, src = _f64(batch.features), _f64(batch.labels), _f64(source_features)
    dm, tmp = _as_device(model, rows=x.shape[0] + src.shape[0])
    loss = C.c_double()
    try:
        _ck(lib().moses_gradients_mmd(dm.h, _p(x), _p(y), x.shape[0], x.shape[1], _p(src), src.shape[0], beta, sigma,
                                      C.byref(loss)))
        g = dm.gradients()
    finally:
        if tmp:
            dm.close()
    return (g, loss.value) if want_loss else g


def adam_update(model: DeviceModel, lr, b1=0.9, b2=0.999, eps=1e-8, step=1, mask: Optional[ParamMask] = None):
    m = None if mask is None else np.ascontiguousarray(mask.transferable, dtype=np.uint8)
    _ck(lib().moses_adam_update(model.h, lr, b1, b2, eps, step, _p(m), 0 if m is None else len(m)))


# ---------------------------------------------------------------- files (model.cpp:344-412, lottery.cpp:182-240)
def serialize(params: CostModelParams) -> bytes:
    d = _dims(params.dims)
    n = lib().moses_serialize(_p(d), len(d), _p(params.params), _p(params.momentum), None, 0)
    if n < 0:
        _ck(int(-n))
    buf = (C.c_uint8 * n)()
    lib().moses_serialize(_p(d), len(d), _p(params.params), _p(params.momentum), C.addressof(buf), n)
    return bytes(buf)


def deserialize(blob: bytes) -> CostModelParams:
    b = np.frombuffer(blob, dtype=np.uint8)
    dims = np.zeros(4, dtype=np.int32)
    cap = max((len(blob) - 12) // 16, 1)
    w = np.zeros(cap)
    m = np.zeros(cap)
    _ck(lib().moses_deserialize(_p(b) if len(b) else None, len(b), _p(dims), _p(w), _p(m), cap))
    return CostModelParams([int(v) for v in dims], w, m)


def save_model(params: CostModelParams, path: str):
    blob = serialize(params)
    try:
        with open(path, "wb") as f:
            f.write(blob)
    except OSError as e:
        raise MosesError(24, f"cannot open {path} for writing") from e


def load_model(path: str) -> CostModelParams:
    try:
        with open(path, "rb") as f:
            blob = f.read()
    except OSError as e:
        raise MosesError(24, f"cannot open model file {path}") from e
    return deserialize(blob)


def write_mask(mask: ParamMask, path: str):
    m = np.ascontiguousarray(mask.transferable, dtype=np.uint8)
    n = lib().moses_write_mask(_p(m), len(m), mask.phase, mask.mode, mask.value, None, 0)
    buf = (C.c_uint8 * n)()
    lib().moses_write_mask(_p(m), len(m), mask.phase, mask.mode, mask.value, C.addressof(buf), n)
    try:
        with open(path, "wb") as f:
            f.write(bytes(buf))
    except OSError as e:
        raise MosesError(24, f"cannot open {path} for writing") from e


def read_mask(path: str) -> ParamMask:
    try:
        with open(path, "rb") as f:
            blob = f.read()
    except OSError as e:
        raise MosesError(24, f"cannot open mask file {path}") from e
    b = np.frombuffer(blob, dtype=np.uint8)
    n = C.c_int64()
    ph = C.c_int32()
    mo = C.c_int32()
    val = C.c_double()
    _ck(lib().moses_read_mask(_p(b), len(b), None, 0, C.byref(n), C.byref(ph), C.byref(mo), C.byref(val)))
    out = np.zeros(n.value, dtype=np.uint8)
    _ck(lib().moses_read_mask(_p(b), len(b), _p(out), len(out), C.byref(n), C.byref(ph), C.byref(mo),
                              C.byref(val)))
    return ParamMask(out.astype(bool), ph.value, mo.value, val.value)


# ---------------------------------------------------------------- candidate generation (space.cpp:140-197)
TEMPLATE_ROLES = {"tile_x": 0, "tile_y": 1, "unroll": 2, "vectorize": 3, "parallel": 4}


def encode_configs_device(task, knobs, first: int, n: int, dtype: int = DTYPE_F32, feat_ptr=None, ld: int = 16,
                          D: int = 16, hash_ptr=None, values_ptr=None):
    """Configs [first, first+n) of enumerate_configs' order, on the device: feature rows (encode_features),
    FNV-1a hashes (config_hash), knob values. task = (work_gflops, bytes_per_unit, ideal_log2_tiles,
    ideal_log2_unroll); knobs = [(name, sorted domain)]; outputs are device pointers (or None)."""
    t = np.ascontiguousarray(task, dtype=np.float64)
    dom = np.ascontiguousarray([v for _, d in knobs for v in d], dtype=np.int64)
    sizes = np.ascontiguousarray([len(d) for _, d in knobs], dtype=np.int32)
    roles = np.ascontiguousarray([TEMPLATE_ROLES.get(k, -1) for k, _ in knobs], dtype=np.int32)
    _ck(lib().moses_encode_configs_device(_p(t), _p(dom), _p(sizes), _p(roles), len(knobs), first, n, dtype,
                                          feat_ptr, ld, D, hash_ptr, values_ptr))


# ---------------------------------------------------------------- simulated hardware (oracle.cpp:33-105)
def _space_arrays(knobs):
    dom = np.ascontiguousarray([v for _, d in knobs for v in d], dtype=np.int64)
    sizes = np.ascontiguousarray([len(d) for _, d in knobs], dtype=np.int32)
    roles = np.ascontiguousarray([TEMPLATE_ROLES.get(k, -1) for k, _ in knobs], dtype=np.int32)
    return dom, sizes, roles


def _device6(device):
    return np.ascontiguousarray([device["peak_gflops"], device["parallel_units"], device["vector_lanes"],
                                 device["cache_bytes"], device["measure_overhead_ms"], device["noise_std"]],
                                dtype=np.float64)


def _task4(task):
    if isinstance(task, dict):
        task = (task["work_gflops"], task["bytes_per_unit"], task["ideal_log2_tiles"], task["ideal_log2_unroll"])
    return np.ascontiguousarray(task, dtype=np.float64)


def measure_configs_device(device, task_id, task, knobs, seed, first, n, clean_ptr=None, thr_ptr=None, lat_ptr=None,
                           wall_ptr=None, label_ptr=None):
    """clean_latency_ms / measure() over configs [first, first+n) into device buffers (pointers or None)."""
    dom, sizes, roles = _space_arrays(knobs)
    _ck(lib().moses_measure_configs_device(_p(_device6(device)), int(device["repeats"]), device["id"].encode(),
                                           task_id.encode(), _p(_task4(task)), _p(dom), _p(sizes), _p(roles),
                                           len(knobs), seed, first, n, clean_ptr, thr_ptr, lat_ptr, wall_ptr,
                                           label_ptr))


def true_best(device, task, knobs):
    """oracle.cpp:90-105 on the device: (values, latency_ms) of the exhaustive noise-free optimum."""
    dom, sizes, roles = _space_arrays(knobs)
    v = np.zeros(len(knobs), dtype=np.int64)
    lat = C.c_double()
    _ck(lib().moses_true_best(_p(_device6(device)), _p(_task4(task)), _p(dom), _p(sizes), _p(roles), len(knobs),
                              _p(v), C.byref(lat)))
    return v.tolist(), lat.value


# ---------------------------------------------------------------- training-data pipeline (data.cpp, tuner.cpp:130-156)
def generate_dataset_device(device, task_id: str, task, knobs, samples: int, seed: int, dtype: int = DTYPE_F32,
                            feat_ptr=None, ld: int = 16, D: int = 16, values_ptr=None, thr_ptr=None, lat_ptr=None,
                            wall_ptr=None, label_ptr=None):
    """generate_dataset (data.cpp:49-65) for one task into device buffers (pointers or None): keyed
    sample_config draws, feature rows, knob values (samples x n_knobs int64), measure() outputs."""
    dom, sizes, roles = _space_arrays(knobs)
    _ck(lib().moses_generate_dataset_device(_p(_device6(device)), int(device["repeats"]), device["id"].encode(),
                                            task_id.encode(), _p(_task4(task)), _p(dom), _p(sizes), _p(roles),
                                            len(knobs), samples, seed, dtype, feat_ptr, ld, D, values_ptr, thr_ptr,
                                            lat_ptr, wall_ptr, label_ptr))


def encode_values_device(task, knobs, values_ptr, n: int, dtype: int = DTYPE_F32, feat_ptr=None, ld: int = 16,
                         D: int = 16, hash_ptr=None):
    """validate_config + encode_features (space.cpp:69-81,140-159) over device rows of knob values.
    Raises MosesError(invalid_config) naming the first bad row."""
    dom, sizes, roles = _space_arrays(knobs)
    bad = C.c_int64(-1)
    _ck(lib().moses_encode_values_device(_p(_task4(task)), _p(dom), _p(sizes), _p(roles), len(knobs), values_ptr, n,
                                         dtype, feat_ptr, ld, D, hash_ptr, C.byref(bad)))


def epoch_seed(seed: int, epoch: int) -> int:
    """KeyBuilder(seed, "epoch", epoch) (tuner.cpp:136-139)."""
    return int(lib().moses_epoch_seed(seed, epoch))


class RankingPlan:
    """make_ranking_batches (data.cpp:128-164) as row indices: batch b = rows[off[b]:off[b+1]] of task
    task_ids[task[b]]."""

    def __init__(self, rows, off, task, task_ids, dropped):
        self.rows, self.off, self.task, self.task_ids, self.dropped_singletons = rows, off, task, task_ids, dropped

    def __len__(self):
        return len(self.off) - 1

    def batch(self, b):
        return self.task_ids[self.task[b]], self.rows[self.off[b]:self.off[b + 1]]


def make_ranking_batches(record_task, task_ids, batch_size: int, seed: int) -> RankingPlan:
    """record_task: per-record index into task_ids (or the task-id strings themselves)."""
    if len(record_task) and isinstance(record_task[0], str):
        ids = list(dict.fromkeys(list(task_ids) + list(record_task)))
        ix = {t: i for i, t in enumerate(ids)}
        record_task, task_ids = [ix[t] for t in record_task], ids
    rt = np.ascontiguousarray(record_task, dtype=np.int32)
    n = len(rt)
    enc = [t.encode() for t in task_ids]
    arr = (C.c_char_p * max(1, len(enc)))(*enc)
    rows = np.zeros(max(n, 1), dtype=np.int64)
    off = np.zeros(n // 2 + 2, dtype=np.int64)
    task = np.zeros(n // 2 + 1, dtype=np.int32)
    nb = C.c_int64()
    dropped = C.c_int64()
    _ck(lib().moses_ranking_plan(_p(rt), n, C.cast(arr, C.c_void_p), len(enc), batch_size, seed, _p(rows), _p(off),
                                 _p(task), C.byref(nb), C.byref(dropped)))
    k = nb.value
    return RankingPlan(rows[:off[k]].copy(), off[:k + 1].copy(), task[:k].copy(), list(task_ids), dropped.value)


def replay_rows(n_records: int, size: int, seed: int) -> np.ndarray:
    """sample_replay_features' row choice (data.cpp:166-183)."""
    out = np.zeros(max(1, min(max(n_records, 0), max(size, 0))), dtype=np.int64)
    k = C.c_int64()
    _ck(lib().moses_replay_rows(n_records, size, seed, _p(out), C.byref(k)))
    return out[:k.value].copy()


def train_plan_device(model, x_ptr, ldx: int, y_ptr, n_records: int, plan: RankingPlan, lr: float,
                      mu: float = 0.9) -> float:
    """One pretrain epoch (tuner.cpp:140-155) over a device-resident packed dataset; returns the mean
    batch loss."""
    rows = np.ascontiguousarray(plan.rows, dtype=np.int64)
    off = np.ascontiguousarray(plan.off, dtype=np.int64)
    out = C.c_double()
    _ck(lib().moses_train_plan_device(model.h, x_ptr, ldx, y_ptr, n_records, _p(rows), _p(off), len(off) - 1, lr, mu,
                                      C.byref(out)))
    return out.value


def pretrain_device(model, x_ptr, ldx: int, y_ptr, record_task, task_ids, batch_size: int = 512, seed: int = 0,
                    epochs: int = 30, lr: float = 0.001, mu: float = 0.9):
    """pretrain (tuner.cpp:130-156) on the device: returns (epoch_mean_loss list, dropped_singletons) like
    PretrainLog. record_task: per-record index into task_ids (or the ids themselves)."""
    if len(record_task) and isinstance(record_task[0], str):
        ids = list(dict.fromkeys(list(task_ids) + list(record_task)))
        ix = {t: i for i, t in enumerate(ids)}
        record_task, task_ids = [ix[t] for t in record_task], ids
    rt = np.ascontiguousarray(record_task, dtype=np.int32)
    enc = [t.encode() for t in task_ids]
    arr = (C.c_char_p * max(1, len(enc)))(*enc)
    losses = np.zeros(max(epochs, 1))
    dropped = C.c_int64()
    _ck(lib().moses_pretrain_device(model.h, x_ptr, ldx, y_ptr, _p(rt), len(rt), C.cast(arr, C.c_void_p), len(enc),
                                    batch_size, seed, epochs, lr, mu, _p(losses), C.byref(dropped)))
    return losses[:epochs].tolist(), dropped.value


def evolve(model, task, knobs, population: int = 128, generations: int = 4, mutation_count: int = 4,
           survivors: int = 32, epsilon_random: float = 0.05, seed: int = 0, lin_w=None):
    """evolve (search.cpp:41-71) with device encoding + scoring by `model` (or, model=None, the linear
    test scorer sum_k lin_w[k] * value_k). Returns (values [n x n_knobs], scores [n]) sorted by
    score desc then configuration asc."""
    dom, sizes, roles = _space_arrays(knobs)
    cap = max(population, survivors * (1 + mutation_count))
    vals = np.zeros((cap, len(knobs)), dtype=np.int64)
    scores = np.zeros(cap)
    n = C.c_int64()
    lw = None if lin_w is None else np.ascontiguousarray(lin_w, dtype=np.float64)
    _ck(lib().moses_evolve(model.h if model is not None else None, _p(lw), _p(_task4(task)), _p(dom), _p(sizes),
                           _p(roles), len(knobs), population, generations, mutation_count, survivors, epsilon_random,
                           seed, _p(vals), _p(scores), cap, C.byref(n)))
    return vals[:n.value], scores[:n.value]


def pretrain(model, tasks, knobs, record_task, values, throughput, batch_size: int = 512, seed: int = 0,
             epochs: int = 30, lr: float = 0.001, mu: float = 0.9):
    """pretrain (tuner.cpp:130-156) from host records on the device. tasks = [(task_id, task4)];
    record_task: per-record index into tasks; values: n x n_knobs; throughput: labels.
    Returns (epoch_mean_loss list, dropped_singletons); the parameters stay on `model`."""
    dom, sizes, roles = _space_arrays(knobs)
    enc = [t.encode() for t, _ in tasks]
    arr = (C.c_char_p * max(1, len(enc)))(*enc)
    t4 = np.ascontiguousarray([_task4(t) for _, t in tasks], dtype=np.float64)
    rt = np.ascontiguousarray(record_task, dtype=np.int32)
    v = np.ascontiguousarray(values, dtype=np.int64)
    thr = np.ascontiguousarray(throughput, dtype=np.float64)
    losses = np.zeros(max(epochs, 1))
    dropped = C.c_int64()
    _ck(lib().moses_pretrain(model.h, len(tasks), C.cast(arr, C.c_void_p), _p(t4), _p(dom), _p(sizes), _p(roles),
                             len(knobs), _p(rt), _p(v), _p(thr), len(rt), batch_size, seed, epochs, lr, mu,
                             _p(losses), C.byref(dropped)))
    return losses[:epochs].tolist(), dropped.value


def pretrain_jobs(models, seeds, x_ptr, ldx: int, y_ptr, record_task, task_ids, batch_size: int = 512,
                  epochs: int = 30, lr: float = 0.001, mu: float = 0.9, threads: int = 0):
    """Independent pretrain runs (one per (model, seed)) over one device-resident dataset on a native
    worker pool (tuner.cpp:331-374). Returns (epoch_mean_loss [jobs x epochs], dropped [jobs])."""
    if len(record_task) and isinstance(record_task[0], str):
        ids = list(dict.fromkeys(list(task_ids) + list(record_task)))
        ix = {t: i for i, t in enumerate(ids)}
        record_task, task_ids = [ix[t] for t in record_task], ids
    rt = np.ascontiguousarray(record_task, dtype=np.int32)
    enc = [t.encode() for t in task_ids]
    arr = (C.c_char_p * max(1, len(enc)))(*enc)
    hs = (C.c_void_p * max(1, len(models)))(*[m.h.value if hasattr(m.h, "value") else m.h for m in models])
    sd = np.ascontiguousarray(seeds, dtype=np.uint64)
    losses = np.zeros((max(len(models), 1), max(epochs, 1)))
    dropped = np.zeros(max(len(models), 1), dtype=np.int64)
    _ck(lib().moses_pretrain_jobs(len(models), C.cast(hs, C.c_void_p), _p(sd), x_ptr, ldx, y_ptr, _p(rt), len(rt),
                                  C.cast(arr, C.c_void_p), len(enc), batch_size, epochs, lr, mu, threads,
                                  _p(losses), _p(dropped)))
    return losses[:len(models), :epochs], dropped[:len(models)]


def pretrain_jobs_mapped(models, seeds, x_ptrs, ldx: int, y_ptrs, record_task, task_ids, batch_size: int = 512,
                         epochs: int = 30, lr: float = 0.001, mu: float = 0.9, threads: int = 0):
    """pretrain_jobs with job j over its own device's copy of the store (x_ptrs[j], y_ptrs[j]): the
    (seed) job grid spread over the GPUs the handles were created on."""
    if len(record_task) and isinstance(record_task[0], str):
        ids = list(dict.fromkeys(list(task_ids) + list(record_task)))
        ix = {t: i for i, t in enumerate(ids)}
        record_task, task_ids = [ix[t] for t in record_task], ids
    rt = np.ascontiguousarray(record_task, dtype=np.int32)
    enc = [t.encode() for t in task_ids]
    arr = (C.c_char_p * max(1, len(enc)))(*enc)
    n = len(models)
    hs = (C.c_void_p * max(1, n))(*[m.h.value if hasattr(m.h, "value") else m.h for m in models])
    xs = (C.c_void_p * max(1, n))(*[int(p.value if hasattr(p, "value") else p) for p in x_ptrs])
    ys = (C.c_void_p * max(1, n))(*[int(p.value if hasattr(p, "value") else p) for p in y_ptrs])
    sd = np.ascontiguousarray(seeds, dtype=np.uint64)
    losses = np.zeros((max(n, 1), max(epochs, 1)))
    dropped = np.zeros(max(n, 1), dtype=np.int64)
    _ck(lib().moses_pretrain_jobs_mapped(n, C.cast(hs, C.c_void_p), _p(sd), C.cast(xs, C.c_void_p), ldx,
                                         C.cast(ys, C.c_void_p), _p(rt), len(rt), C.cast(arr, C.c_void_p), len(enc),
                                         batch_size, epochs, lr, mu, threads, _p(losses), _p(dropped)))
    return losses[:n, :epochs], dropped[:n]


class RecordStore:
    """Line-delimited measurement records (data.cpp:67-126) held by the native reader."""

    def __init__(self, handle=None):
        self.h = C.c_void_p(handle)
        if handle is None:
            _ck(lib().moses_records_create(C.byref(self.h)))

    @classmethod
    def read(cls, path: str) -> "RecordStore":
        h = C.c_void_p()
        _ck(lib().moses_records_read(path.encode(), C.byref(h)))
        return cls(h.value)

    def __del__(self):
        if getattr(self, "h", None) and self.h.value and _lib is not None:
            _lib.moses_records_destroy(self.h)
            self.h = C.c_void_p()

    def append(self, task_id: str, device_id: str, values, throughput, latency, wall_cost, seq):
        v = np.ascontiguousarray(values, dtype=np.int64)
        if v.ndim == 1:
            v = v.reshape(1, -1)
        n = v.shape[0]
        cols = [np.ascontiguousarray(np.broadcast_to(a, (n,)), dtype=t)
                for a, t in ((throughput, np.float64), (latency, np.float64), (wall_cost, np.float64),
                             (seq, np.uint64))]
        _ck(lib().moses_records_append(self.h, task_id.encode(), device_id.encode(), n, v.shape[1], _p(v),
                                       *(_p(c) for c in cols)))

    def write(self, path: str):
        _ck(lib().moses_records_write(self.h, path.encode()))

    def shape(self):
        n, nv, nt, nd = C.c_int64(), C.c_int64(), C.c_int32(), C.c_int32()
        _ck(lib().moses_records_shape(self.h, C.byref(n), C.byref(nv), C.byref(nt), C.byref(nd)))
        return n.value, nv.value, nt.value, nd.value

    def __len__(self):
        return self.shape()[0]

    def task_ids(self):
        return [lib().moses_records_task_id(self.h, t).decode() for t in range(self.shape()[2])]

    def device_ids(self):
        return [lib().moses_records_device_id(self.h, d).decode() for d in range(self.shape()[3])]

    def export(self, pinned: bool = False):
        """Flat arrays: task (int32 index into task_ids()), device, value_off, values, throughput,
        latency, wall_cost, seq. pinned=True returns page-locked torch tensors (ready for a
        non-blocking upload)."""
        n, nv, _, _ = self.shape()
        specs = [("task", n, np.int32), ("device", n, np.int32), ("value_off", n + 1, np.int64),
                 ("values", nv, np.int64), ("throughput", n, np.float64), ("latency", n, np.float64),
                 ("wall_cost", n, np.float64), ("seq", n, np.uint64)]
        if pinned:
            import torch
            tmap = {np.int32: torch.int32, np.int64: torch.int64, np.float64: torch.float64, np.uint64: torch.int64}
            out = {k: torch.empty(max(m, 1), dtype=tmap[t], pin_memory=True) for k, m, t in specs}
            ptrs = [out[k].data_ptr() for k, _, _ in specs]
            _ck(lib().moses_records_export(self.h, *ptrs))
            return {k: out[k][:m] for k, m, _ in specs}
        out = {k: np.zeros(max(m, 1), dtype=t) for k, m, t in specs}
        _ck(lib().moses_records_export(self.h, *(_p(out[k]) for k, _, _ in specs)))
        return {k: out[k][:m] for k, m, _ in specs}


# ---------------------------------------------------------------- online tuning
STRATEGY_RAW, STRATEGY_RANDOM_INIT, STRATEGY_PRETRAIN_ONLY, STRATEGY_VANILLA, STRATEGY_MOSES = 0, 1, 2, 3, 4


class _DeviceSpec(C.Structure):
    _fields_ = [("id", C.c_char_p), ("params", C.c_double * 6), ("repeats", C.c_int32)]


class _TaskSpec(C.Structure):
    _fields_ = [("id", C.c_char_p), ("task4", C.c_double * 4), ("domains", C.c_void_p), ("domain_sizes", C.c_void_p),
                ("roles", C.c_void_p), ("n_knobs", C.c_int32)]


class _TuneBudget(C.Structure):
    _fields_ = [("trials_per_task", C.c_int32), ("train_fraction", C.c_double), ("num_batches", C.c_int32),
                ("cv_threshold", C.c_double), ("population", C.c_int32), ("generations", C.c_int32),
                ("mutation_count", C.c_int32), ("survivors", C.c_int32), ("epsilon_random", C.c_double),
                ("learning_rate", C.c_double), ("weight_decay", C.c_double), ("adversary_beta", C.c_double),
                ("lottery_mode", C.c_int32), ("lottery_value", C.c_double), ("adversary", C.c_int32),
                ("replay_size", C.c_int32)]


class _TaskResult(C.Structure):
    _fields_ = [("capacity", C.c_int64), ("values", C.c_void_p), ("throughput", C.c_void_p), ("latency", C.c_void_p),
                ("wall_cost", C.c_void_p), ("n_records", C.c_int64), ("best_values", C.c_void_p),
                ("best_latency_ms", C.c_double), ("wall_cost_ms", C.c_double), ("batch_means", C.c_void_p),
                ("cvs", C.c_void_p), ("n_batch_means", C.c_int32), ("termination_batch", C.c_int32),
                ("measured_trials", C.c_int32), ("prediction_trials", C.c_int32), ("unspent_trials", C.c_int32),
                ("predicted_scores", C.c_void_p)]


@dataclass
class TuneBudget:  # tuner.hpp TuneBudget with the reference defaults (search.hpp, model.hpp, tuner.hpp)
    trials_per_task: int = 64
    train_fraction: float = 0.9
    num_batches: int = 5
    cv_threshold: float = 0.05
    population: int = 128
    generations: int = 4
    mutation_count: int = 4
    survivors: int = 32
    epsilon_random: float = 0.05
    learning_rate: float = 0.001
    weight_decay: float = 0.01
    adversary_beta: float = 0.01
    lottery_mode: int = RATIO
    lottery_value: float = 0.5
    adversary: bool = True
    replay_size: int = 256

    def _c(self):
        return _TuneBudget(self.trials_per_task, self.train_fraction, self.num_batches, self.cv_threshold,
                           self.population, self.generations, self.mutation_count, self.survivors,
                           self.epsilon_random, self.learning_rate, self.weight_decay, self.adversary_beta,
                           self.lottery_mode, self.lottery_value, int(self.adversary), self.replay_size)


@dataclass
class TaskResult:  # tuner.hpp TaskResult + ControllerTrace
    values: np.ndarray
    throughput: np.ndarray
    latency: np.ndarray
    wall_cost: np.ndarray
    best_values: np.ndarray
    best_latency_ms: float
    wall_cost_ms: float
    batch_means: np.ndarray
    cvs: np.ndarray
    termination_batch: int
    measured_trials: int
    prediction_trials: int
    unspent_trials: int
    predicted_scores: np.ndarray


def _c_device(device):
    d = _DeviceSpec()
    d.id = device["id"].encode()
    d.params[:] = list(_device6(device))
    d.repeats = int(device["repeats"])
    return d


def _c_task(task_id, task, knobs, keep):
    dom, sizes, roles = _space_arrays(knobs)
    keep += [dom, sizes, roles]
    t = _TaskSpec()
    t.id = task_id.encode()
    t.task4[:] = list(_task4(task))
    t.domains, t.domain_sizes, t.roles, t.n_knobs = dom.ctypes.data, sizes.ctypes.data, roles.ctypes.data, len(knobs)
    return t


def _alloc_result(budget: TuneBudget, nk: int):
    cap = max(1, budget.trials_per_task)
    arrs = {"values": np.zeros((cap, nk), dtype=np.int64), "throughput": np.zeros(cap), "latency": np.zeros(cap),
            "wall_cost": np.zeros(cap), "best_values": np.zeros(nk, dtype=np.int64),
            "batch_means": np.zeros(max(1, budget.num_batches)), "cvs": np.zeros(max(1, budget.num_batches)),
            "predicted_scores": np.zeros(cap)}
    r = _TaskResult()
    r.capacity = cap
    for k, a in arrs.items():
        setattr(r, k, a.ctypes.data)
    return r, arrs


def _result(r, arrs):
    n, nb = r.n_records, r.n_batch_means
    return TaskResult(arrs["values"][:n].copy(), arrs["throughput"][:n].copy(), arrs["latency"][:n].copy(),
                      arrs["wall_cost"][:n].copy(), arrs["best_values"].copy(), r.best_latency_ms, r.wall_cost_ms,
                      arrs["batch_means"][:nb].copy(), arrs["cvs"][:nb].copy(), r.termination_batch,
                      r.measured_trials, r.prediction_trials, r.unspent_trials,
                      arrs["predicted_scores"][:r.prediction_trials].copy())


def tune_task(model: DeviceModel, strategy: int, device, task_id: str, task, knobs, budget: TuneBudget, seed: int,
              source_features=None) -> TaskResult:
    """tune_task (tuner.cpp:158-286) on the parameters of `model` (updated in place)."""
    keep = []
    t = _c_task(task_id, task, knobs, keep)
    r, arrs = _alloc_result(budget, len(knobs))
    src = None if source_features is None else np.ascontiguousarray(source_features, dtype=np.float64)
    _ck(lib().moses_tune_task(model.h, strategy, C.byref(_c_device(device)), C.byref(t), C.byref(budget._c()), seed,
                              _p(src), 0 if src is None else src.shape[0], C.byref(r)))
    return _result(r, arrs)


def tune_jobs(models, strategies, seeds, task_of, tasks, knobs, device, budget: TuneBudget, source_features=None,
              threads: int = 0):
    """The (strategy, seed, task) job grid (tuner.cpp:307-374): job j on models[j]; tasks = [(task_id, task)],
    every task over the same knob template. Returns [TaskResult]."""
    keep = []
    n = len(models)
    ts = (_TaskSpec * max(1, len(tasks)))(*[_c_task(tid, t, knobs, keep) for tid, t in tasks])
    res = [_alloc_result(budget, len(knobs)) for _ in range(n)]
    rs = (_TaskResult * max(1, n))(*[r for r, _ in res])
    hs = (C.c_void_p * max(1, n))(*[m.h for m in models])
    st = np.ascontiguousarray(strategies, dtype=np.int32)
    sd = np.ascontiguousarray(seeds, dtype=np.uint64)
    to = np.ascontiguousarray(task_of, dtype=np.int32)
    src = None if source_features is None else np.ascontiguousarray(source_features, dtype=np.float64)
    _ck(lib().moses_tune_jobs(n, C.cast(hs, C.c_void_p), _p(st), _p(sd), _p(to), C.cast(ts, C.c_void_p), len(tasks),
                              C.byref(_c_device(device)), C.byref(budget._c()), _p(src),
                              0 if src is None else src.shape[0], threads, C.cast(rs, C.c_void_p)))
    return [_result(rs[j], res[j][1]) for j in range(n)]
