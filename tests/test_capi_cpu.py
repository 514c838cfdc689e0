"""The C-ABI library loads and exports every symbol include/tem.h declares; host-only
sizing functions behave (no compute calls: there is no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "tem.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s+\*?([a-z_][a-z0-9_]*)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n not in ("if", "while")))


def test_header_declares_the_boundary():
    names = header_functions()
    for n in ("tem_init", "tem_step", "ring_allreduce", "tem_shutdown"):
        assert n in names
    assert len(names) >= 15


def test_library_exports_every_symbol():
    from paper_1906_06496_b200 import tem
    L = tem.lib()
    for n in header_functions():
        assert hasattr(L, n), n
    assert set(header_functions()) <= set(tem.EXPORTS) | {"tem_status_string"}


def base_cfg(tem, N=8, B=16, prec=0):
    c = tem.tem_config()
    c.world_size, c.rank, c.local_ranks = N, 0, 1
    c.batch_per_rank, c.seq_len, c.c_in, c.c_hidden, c.c_out = B, 100, 400, 512, 3
    c.precision, c.lr = prec, 0.01
    return c


def test_sizes():
    from paper_1906_06496_b200 import tem
    for N, kp in ((1, 1403396), (2, 1403400), (4, 1403408), (8, 1403424)):
        c = base_cfg(tem, N)
        assert tem.tem_num_params(c) == 1403395
        assert tem.tem_kpad(c, 1403395) == kp
        assert tem.tem_sym_user_offset(c) >= 4 * kp
        assert tem.tem_sym_bytes(c) > tem.tem_sym_user_offset(c) + 4 * kp
        assert tem.tem_workspace_bytes(c) > 0
    # the fp32 path adds the four lo residual planes (x, h1, dA2, dA1) and the weights' lo copy
    assert tem.tem_workspace_bytes(base_cfg(tem, 8, 256, 1)) < tem.tem_workspace_bytes(base_cfg(tem, 8, 256, 0))


@pytest.mark.parametrize("field,value", [("world_size", 0), ("world_size", 9), ("rank", 8),
                                         ("c_out", 2), ("c_in", 401), ("c_hidden", 100),
                                         ("precision", 2), ("lr", -1.0), ("batch_per_rank", -1),
                                         ("local_ranks", 3)])
def test_invalid_configs_rejected(field, value):
    from paper_1906_06496_b200 import tem
    c = base_cfg(tem)
    setattr(c, field, value)
    assert tem.tem_num_params(c) == 0
    assert tem.tem_workspace_bytes(c) == 0
    ctx = ctypes.c_void_p()
    assert tem.lib().tem_init(ctypes.byref(c), None, ctypes.byref(ctx)) == tem.TEM_ERR_INVALID_ARG
    assert not ctx.value


@pytest.mark.parametrize("fields", [dict(optimizer=3), dict(optimizer=1, beta1=1.0, beta2=0.999, eps=1e-8),
                                    dict(optimizer=1, beta1=0.9, beta2=-0.1, eps=1e-8),
                                    dict(optimizer=1, beta1=0.9, beta2=0.999, eps=0.0),
                                    dict(optimizer=2, momentum=1.0), dict(optimizer=2, momentum=-0.5),
                                    dict(exchange_buckets=3), dict(exchange_buckets=2, exchange=1)])
def test_invalid_optimizer_rejected(fields):
    from paper_1906_06496_b200 import tem
    c = base_cfg(tem)
    for k, v in fields.items():
        setattr(c, k, v)
    assert tem.tem_num_params(c) == 0


def test_adam_workspace_holds_moments():
    """Adam adds m and v ([K_pad] fp32 each) and beta^t to every rank's workspace (reading R22)."""
    from paper_1906_06496_b200 import tem
    c = base_cfg(tem, 2)
    sgd = tem.tem_workspace_bytes(c)
    c.optimizer, c.beta1, c.beta2, c.eps = tem.TEM_OPT_ADAM, 0.9, 0.999, 1e-8
    assert tem.tem_num_params(c) == 1403395
    assert tem.tem_workspace_bytes(c) - sgd >= 2 * 4 * tem.tem_kpad(c, 1403395)


def test_pgm_rejects_bad_shapes():
    """tem_pgm validates before touching the GPU (T <= 128, P >= 1; B = 0 is a no-op)."""
    from paper_1906_06496_b200 import tem
    L = tem.lib()
    nul = [None] * 9
    assert L.tem_pgm(1, 129, 0, 4, *nul) == tem.TEM_ERR_INVALID_ARG
    assert L.tem_pgm(1, 10, 0, 0, *nul) == tem.TEM_ERR_INVALID_ARG
    assert L.tem_pgm(1, 10, 0, 4, *nul) == tem.TEM_ERR_INVALID_ARG
    assert L.tem_pgm(0, 10, 0, 4, *nul) == tem.TEM_OK


def test_null_context_calls():
    from paper_1906_06496_b200 import tem
    L = tem.lib()
    assert L.tem_shutdown(None) == tem.TEM_OK
    assert L.tem_step(None, None, None, None, None) == tem.TEM_ERR_STATE
    assert L.ring_allreduce(None, None, 10, 0, None) == tem.TEM_ERR_STATE
    assert tem.status_string(tem.TEM_ERR_PROTOCOL) == "TEM_ERR_PROTOCOL"


def test_product_does_not_touch_oracle():
    """The product package never imports / links the oracle."""
    pkg = os.path.join(ROOT, "paper_1906_06496_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "tem_oracle" not in txt, f
