"""B200-native engine for the Student Parallelism hot path (arXiv 2408.12526).

K flat students run concurrently on every request and their alpha-weighted outputs are summed
into logits through one shared classifier (EnsembleState.rep + classifier, distill.py:169-178,
:512). The hot path is hand-written sm_100a CUDA behind a C ABI (include/studentpar_b200.h);
this package is the Python host that mirrors the reference's object API.
"""
from .weights import (  # noqa: F401
    PRESETS,
    BertConfig,
    BertGroupWeights,
    DenseGroupWeights,
    dense_group_from_arrays,
    dense_group_from_ensemble,
    random_bert_group,
    random_dense_group,
)

__version__ = "0.1.0"


def __getattr__(name):
    # torch-dependent pieces are imported lazily so the weight/config layer stays importable anywhere
    if name == "StudentGroup":
        from .group import StudentGroup

        return StudentGroup
    raise AttributeError(name)
