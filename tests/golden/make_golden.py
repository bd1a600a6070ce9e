"""Generate the golden fixtures of tests/golden/ from the UNMODIFIED reference package.

Run in the build container (the reference is importable only there):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (small, committed; they travel to the GPU box where the reference does not exist):
  dense_ref_<name>.npz    reference StudentModel groups built with the reference's own
                          constructors, inputs, and the reference's rep / logits / argmax for
                          every prefix k (EnsembleState.rep distill.py:169-178, :512-513)
  ensemble_trained.json   a group trained by the reference (sequential_training +
                          adaptive_pruning on make_gaussian_task), saved with save_ensemble
                          (ensemble-checkpoint-v1, binary mode, bit exact)
  ensemble_trained_task.npz  its validation/test inputs + labels and the reference's
                          prefix_accuracy for every k (real-data argmax parity)
  training_eval_ref.npz   training-side evaluation of that checkpoint by the reference: a trained
                          teacher's reps/logits/head on the validation split, residual_mse for every
                          k (distill.py:297-302), the accumulate_prefix_gradients total (:471-494)
                          and ensemble_accuracy_via_teacher_head (:676-683)
  servesim_ref.npz        generate_workload / allocate_students / nearest_rank_percentile /
                          decide_controller_action reference outputs (serving-side restatements)
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from studentpar import distill as dst  # noqa: E402
from studentpar import nnkernel as nn  # noqa: E402
from studentpar import servesim as ss  # noqa: E402

OUT = Path(__file__).resolve().parent


def make_rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def dense_case(name, d_in, rep_dim, depth, k_students, n_classes, n_rows, seed, alphas=None, engine_precision=False):
    """engine_precision: round matrices + inputs to fp16 and vectors to fp32 BEFORE the reference
    runs, so the fixture holds exactly the values the CUDA engine consumes (stored compactly)."""
    rng = make_rng(seed)
    students = [nn.StudentModel.build(d_in, rep_dim, depth, rng) for _ in range(k_students)]
    mat = (lambda a: a.astype(np.float16).astype(np.float64)) if engine_precision else (lambda a: a)
    vec = (lambda a: a.astype(np.float32).astype(np.float64)) if engine_precision else (lambda a: a)
    for s in students:  # trained groups have nonzero biases; exercise the bias path
        for lay in [s.input_proj, *s.layers]:
            lay.weight[...] = mat(lay.weight)
            lay.bias[...] = vec(rng.normal(0.0, 0.1, size=lay.bias.shape))
    if alphas is None:
        alphas = [1.0] + [float(v) for v in vec(rng.uniform(-0.5, 1.0, size=k_students - 1))]
    clf = nn.DenseLayer.init(n_classes, rep_dim, nn.IDENTITY, rng)
    clf.weight[...] = vec(clf.weight)
    clf.bias[...] = vec(rng.normal(0.0, 0.1, size=n_classes))
    state = dst.EnsembleState(students, alphas, clf)
    x = mat(rng.normal(size=(n_rows, d_in)))
    store_m = (lambda a: a.astype(np.float16)) if engine_precision else (lambda a: a)
    store_v = (lambda a: a.astype(np.float32)) if engine_precision else (lambda a: a)
    arrays = {"x": store_m(x), "alphas": np.asarray(alphas), "w_cls": store_v(clf.weight), "b_cls": store_v(clf.bias)}
    for m, s in enumerate(students):
        arrays[f"s{m}_w_in"] = store_m(s.input_proj.weight)
        arrays[f"s{m}_b_in"] = store_v(s.input_proj.bias)
        for l, lay in enumerate(s.layers):
            arrays[f"s{m}_w{l}"] = store_m(lay.weight)
            arrays[f"s{m}_b{l}"] = store_v(lay.bias)
    for k in range(1, k_students + 1):
        rep = state.rep(x, k)
        logits = state.classifier.forward(rep)
        arrays[f"rep_k{k}"] = rep
        arrays[f"logits_k{k}"] = logits
        arrays[f"pred_k{k}"] = np.argmax(logits, axis=1)
        # 1-D input convention (nnkernel.py:67-70): one sample, squeezed output
        arrays[f"rep1_k{k}"] = state.rep(x[0], k)
    # mid tap of student 0 (nnkernel.py:280-283)
    arrays["mid0"] = students[0].forward(x)[1]
    np.savez_compressed(OUT / f"dense_ref_{name}.npz", depth=depth, k_students=k_students,
                        engine_precision=engine_precision, **arrays)


def trained_case():
    splits = dst.make_gaussian_task(n_classes=2, d_in=8, n_train=160, n_val=96, n_test=96, class_sep=2.5, seed=3)
    teacher = nn.TeacherModel.build(8, 16, 24, 3, 2, make_rng(3))
    dst.train_teacher(teacher, splits, epochs=40, learning_rate=3e-3, seed=3)
    cfg = dst.DistillConfig(max_students=4, epochs_per_student=30, batch_size=32, learning_rate=3e-3,
                            pruning_epochs=15, seed=3)
    state, _records = dst.sequential_training(teacher, splits, cfg)
    state, table, best_k = dst.adaptive_pruning(teacher, state, splits, cfg)
    path = OUT / "ensemble_trained.json"
    dst.save_ensemble(state, path)
    k_max = len(state)
    acc_val = [dst.prefix_accuracy(state, splits.validation, k) for k in range(1, k_max + 1)]
    acc_test = [dst.prefix_accuracy(state, splits.test, k) for k in range(1, k_max + 1)]
    logits = {f"logits_val_k{k}": state.classifier.forward(state.rep(splits.validation.inputs, k))
              for k in range(1, k_max + 1)}
    np.savez_compressed(OUT / "ensemble_trained_task.npz", x_val=splits.validation.inputs,
                        y_val=splits.validation.labels, x_test=splits.test.inputs, y_test=splits.test.labels,
                        acc_val=np.asarray(acc_val), acc_test=np.asarray(acc_test), best_k=best_k, **logits)


def training_eval_case():
    splits = dst.make_gaussian_task(n_classes=2, d_in=8, n_train=160, n_val=96, n_test=96, class_sep=2.5, seed=3)
    teacher = nn.TeacherModel.build(8, 16, 24, 3, 2, make_rng(3))
    dst.train_teacher(teacher, splits, epochs=40, learning_rate=3e-3, seed=3)
    state = dst.load_ensemble(OUT / "ensemble_trained.json")
    val = splits.validation
    t_rep, t_logits = teacher.forward(val.inputs)
    out = {"x_val": val.inputs, "y_val": val.labels, "teacher_rep": t_rep, "teacher_logits": t_logits,
           "head_w": teacher.head.weight, "head_b": teacher.head.bias}
    out["residual_mse"] = np.asarray([dst.residual_mse(teacher, state, val, k) for k in range(1, len(state) + 1)])
    for temp in (1.0, 2.0):
        _, total = dst.accumulate_prefix_gradients(state, val.inputs, t_logits, temp)
        out[f"prefix_total_T{temp:g}"] = np.asarray(total)
    out["acc_teacher_head"] = np.asarray(dst.ensemble_accuracy_via_teacher_head(teacher, state, val))
    np.savez_compressed(OUT / "training_eval_ref.npz", **out)


def servesim_case():
    out = {}
    reqs = ss.generate_workload(ss.PoissonSpec(rps=2000.0, duration_ms=50.0), seed=7)
    out["wl_arrival"] = np.asarray([r.arrival_ms for r in reqs])
    out["wl_len"] = np.asarray([r.length_tokens for r in reqs])
    reqs2 = ss.generate_workload(ss.PoissonSpec(rps=500.0, duration_ms=100.0), seed=1, max_len=512, bin_width=32)
    out["wl2_arrival"] = np.asarray([r.arrival_ms for r in reqs2])
    out["wl2_len"] = np.asarray([r.length_tokens for r in reqs2])
    # bursty phases exactly as cli.py:191-202 builds them (simulate.json phase shape, scaled down)
    from studentpar.seeding import fork_seed
    phased, offset = [], 0.0
    for i, (rps, dur) in enumerate([(2000.0, 40.0), (10000.0, 25.0), (2000.0, 60.0)]):
        part = ss.generate_workload(ss.PoissonSpec(rps=rps, duration_ms=dur), fork_seed(11, f"workload-phase-{i}"))
        phased.extend((r.arrival_ms + offset, r.length_tokens) for r in part)
        offset += dur
    out["ph_arrival"] = np.asarray([a for a, _ in phased])
    out["ph_len"] = np.asarray([n for _, n in phased])
    out["fork_seed_0_x"] = np.asarray([fork_seed(0, "x"), fork_seed(12345, "bert-student-7")], dtype=np.uint64)
    alloc = ss.allocate_students(group_size=3, gpus=4, replicas_per_gpu=3)
    out["alloc_keys"] = np.asarray(sorted(alloc.keys()))
    out["alloc_vals"] = np.asarray([alloc[k] for k in sorted(alloc.keys())])
    vals = list(make_rng(5).normal(10.0, 3.0, size=101))
    out["pct_values"] = np.asarray(vals)
    out["pct_p"] = np.asarray([1.0, 50.0, 95.0, 99.0, 100.0])
    out["pct_out"] = np.asarray([ss.nearest_rank_percentile(vals, p) for p in out["pct_p"]])
    cases = []
    for k in (1, 2, 3, 8):
        for full in (False, True):
            for idle in (None, 0.0, 50.0, 200.0):
                for idle_s, occ_s in ((5, 2), (1, 4), (3, 3)):
                    act = ss.decide_controller_action(k, 1, 8, full, idle, idle_s, occ_s, 100.0)
                    cases.append((k, int(full), -1.0 if idle is None else idle, idle_s, occ_s,
                                  {"drop_one": 0, "add_one": 1, "hold": 2}[act]))
    out["ctrl_cases"] = np.asarray(cases, dtype=np.float64)
    np.savez_compressed(OUT / "servesim_ref.npz", **out)


def main():
    dense_case("tiny", d_in=4, rep_dim=6, depth=2, k_students=3, n_classes=2, n_rows=24, seed=1)
    dense_case("pad", d_in=70, rep_dim=130, depth=3, k_students=3, n_classes=3, n_rows=40, seed=2,
               engine_precision=True)
    dense_case("wide", d_in=64, rep_dim=256, depth=2, k_students=3, n_classes=2, n_rows=32, seed=3,
               engine_precision=True)
    if "--training-eval-only" not in sys.argv:
        trained_case()
    training_eval_case()
    if "--training-eval-only" not in sys.argv:
        servesim_case()
    meta = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/pkg/src/studentpar",
            "numpy": np.__version__}
    (OUT / "golden_meta.json").write_text(json.dumps(meta, indent=1) + "\n")
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
