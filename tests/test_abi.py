"""CPU-side checks of the C ABI: the library loads without a GPU, exports exactly what
include/rlvla.h declares, host-only calls work, and argument validation rejects bad calls
before touching the device."""
import ctypes

import pytest

from paper_2602_05765_b200 import _abi as A


@pytest.fixture(scope="module")
def L():
    from paper_2602_05765_b200 import build
    build.build()
    return A.lib()


def test_exports_every_header_symbol(L):
    names = A.header_functions()
    assert len(names) == 19
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(A._SIGS)


def test_host_only_calls(L):
    assert L.rlvla_abi_version() == 2
    assert L.rlvla_set_reserved_sms(2) == 0 and L.rlvla_set_reserved_sms(0) == 2
    assert L.rlvla_nccl_version() >= 22800
    for s in range(6):
        assert L.rlvla_status_string(s)
    small = L.rlvla_workspace_bytes(0, 1, 1)
    big = L.rlvla_workspace_bytes(0, 4096, 64)
    assert big - small >= 4096 * 4 - 256 and small > 256 * 1024


def test_struct_layouts_match_header(tmp_path):
    """sizeof/offsetof of every ABI struct as the C compiler lays it out == the ctypes mirror."""
    import subprocess
    structs = {"rlvla_traj_buffer": A.c_traj_buffer, "rlvla_step_batch": A.c_step_batch,
               "rlvla_adv_params": A.c_adv_params, "rlvla_logits": A.c_logits,
               "rlvla_ppo_args": A.c_ppo_args, "rlvla_batch_queue": A.c_batch_queue,
               "rlvla_gauss_chain": A.c_gauss_chain}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "rlvla.h"', "int main(void){"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for fname, _ in cls._fields_:
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", A.os.path.dirname(A.HEADER), str(src), "-o", str(exe)], check=True)
    out = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                        check=True).stdout.split("\n") if l)
    for cname, cls in structs.items():
        assert int(out[cname]) == ctypes.sizeof(cls), cname
        for fname, _ in cls._fields_:
            assert int(out[f"{cname}.{fname}"]) == getattr(cls, fname).offset, (cname, fname)


FAKE = 0x10000  # never dereferenced: validation fails before any device work


def _buf(**kw):
    b = A.c_traj_buffer(4, 8, 3, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE)
    for k, v in kw.items():
        setattr(b, k, v)
    return b


def _rec(n=4):
    return A.c_step_batch(n, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE)


def test_scatter_validation(L):
    b, r = _buf(), _rec()
    assert L.rlvla_scatter_steps(None, ctypes.byref(r), 1, 1, FAKE, None) == A.ERR_INVALID_ARG
    assert L.rlvla_scatter_steps(ctypes.byref(_buf(slot_key=None)), ctypes.byref(r), 1, 1, FAKE, None) == A.ERR_INVALID_ARG
    assert L.rlvla_scatter_steps(ctypes.byref(_buf(slot_key=FAKE + 4)), ctypes.byref(r), 1, 1, FAKE, None) == A.ERR_INVALID_ARG
    assert L.rlvla_scatter_steps(ctypes.byref(b), ctypes.byref(r), -1, 1, FAKE, None) == A.ERR_INVALID_ARG
    assert L.rlvla_scatter_steps(ctypes.byref(b), ctypes.byref(r), 1 << 23, 1, FAKE, None) == A.ERR_INVALID_ARG
    assert L.rlvla_scatter_steps(ctypes.byref(b), ctypes.byref(r), 1, 0, FAKE, None) == A.ERR_INVALID_ARG
    assert L.rlvla_scatter_steps(ctypes.byref(b), ctypes.byref(r), 1, (1 << 40) - 2, FAKE, None) == A.ERR_INVALID_ARG
    assert L.rlvla_scatter_steps(ctypes.byref(b), ctypes.byref(r), 1, 1, None, None) == A.ERR_INVALID_ARG
    assert L.rlvla_scatter_steps(ctypes.byref(b), ctypes.byref(_rec(0)), 1, 1, FAKE, None) == A.OK


def test_advantages_validation(L):
    b = _buf()
    p = A.c_adv_params(A.ADV_GAE, 0.99, 0.95, 0, 1e-8, None, 0, 1, 1e-6, 0, 4, 100, 1)
    ws_n = L.rlvla_workspace_bytes(0, 4, 8)
    call = lambda **kw: L.rlvla_advantages(ctypes.byref(kw.get("b", b)), None, ctypes.byref(kw.get("p", p)),  # noqa: E731
                                           kw.get("adv", FAKE), kw.get("ret", FAKE), FAKE,
                                           kw.get("ws", 0x100000), kw.get("wn", ws_n), None, None)
    assert call(adv=None) == A.ERR_INVALID_ARG
    assert call(ret=None) == A.ERR_INVALID_ARG               # GAE needs ret
    assert call(wn=ws_n - 1) == A.ERR_INVALID_ARG
    assert call(ws=0x100010) == A.ERR_INVALID_ARG            # misaligned workspace
    bad = A.c_adv_params(*[getattr(p, f) for f, _ in A.c_adv_params._fields_])
    bad.n_env_global = 8                                      # single rank must equal n_env
    assert call(p=bad) == A.ERR_INVALID_ARG
    g = A.c_adv_params(*[getattr(p, f) for f, _ in A.c_adv_params._fields_])
    g.mode, g.group_size = A.ADV_GRPO, 0
    assert call(p=g) == A.ERR_INVALID_ARG                     # GRPO needs groups
    g.mode = 7
    assert call(p=g) == A.ERR_INVALID_ARG


def test_logprob_validation(L):
    x = A.c_logits(FAKE, A.BF16, 16, 32000, 32000)
    f = A.c_ppo_args(FAKE, None, FAKE, FAKE, FAKE, 7, 100, 1, 0.2, 0.2, 0.0, 0.0, None, None, None)
    call = lambda **kw: L.rlvla_logprob_fwd_bwd(ctypes.byref(kw.get("x", x)), kw.get("t", FAKE),  # noqa: E731
                                                kw.get("logp", FAKE), kw.get("lse", None),
                                                kw.get("g", None), kw.get("f", None),
                                                kw.get("dx", None), kw.get("stats", None),
                                                kw.get("ws", None), kw.get("wn", 0), None, None)
    assert call(t=None) == A.ERR_INVALID_ARG
    assert call(x=A.c_logits(FAKE, 5, 16, 32000, 32000)) == A.ERR_INVALID_ARG
    assert call(x=A.c_logits(FAKE, A.BF16, 16, 32000, 31999)) == A.ERR_INVALID_ARG
    assert call(logp=None) == A.ERR_INVALID_ARG
    assert call(g=FAKE) == A.ERR_INVALID_ARG                  # external bwd needs lse + dlogits
    assert call(f=ctypes.byref(f)) == A.ERR_INVALID_ARG       # no N and no adv_stats
    f.tok_denominator = 10.0
    assert call(f=ctypes.byref(f), g=FAKE, lse=FAKE, dx=FAKE) == A.ERR_INVALID_ARG  # both modes
    f.a_tok = 5
    assert call(f=ctypes.byref(f)) == A.ERR_INVALID_ARG       # rows % a_tok != 0
    f.a_tok = 8
    assert call(f=ctypes.byref(f), stats=FAKE) == A.ERR_INVALID_ARG  # stats need a workspace
    assert call(x=A.c_logits(FAKE, A.BF16, 0, 32000, 32000)) == A.OK  # empty input is a no-op


def test_ppo_loss_validation(L):
    f = A.c_ppo_args(FAKE, None, FAKE, FAKE, FAKE, 4, 100, 1, 0.2, 0.2, 0.0, 1.0, None, None, None)
    assert L.rlvla_ppo_loss(None, 8, None, ctypes.byref(f), FAKE, None, None, None, 0, None, None) == A.ERR_INVALID_ARG
    assert L.rlvla_ppo_loss(FAKE, 8, None, ctypes.byref(f), None, None, None, None, 0, None, None) == A.ERR_INVALID_ARG
    assert L.rlvla_ppo_loss(FAKE, 6, None, ctypes.byref(f), FAKE, None, None, None, 0, None, None) == A.ERR_INVALID_ARG
    f.eps_low = 1.5
    assert L.rlvla_ppo_loss(FAKE, 8, None, ctypes.byref(f), FAKE, None, None, None, 0, None, None) == A.ERR_INVALID_ARG
    f.eps_low = 0.2
    # chunk ratio (R21): a KL term has no step-level reading; accumulate needs N_steps up front
    f.ratio_level, f.logp_ref, f.kl_coef = 1, FAKE, 0.1
    ws_n = L.rlvla_workspace_bytes(0, 1, 1)
    call = lambda: L.rlvla_ppo_loss(FAKE, 8, None, ctypes.byref(f), FAKE, None, None, 0x100000, ws_n, None, None)  # noqa: E731
    assert call() == A.ERR_UNSUPPORTED
    f.kl_coef, f.tok_denominator, f.accumulate = 0.0, 0.0, 1
    assert call() == A.ERR_INVALID_ARG
    # rows = 0 without stats is a no-op even with NULL arrays (a rank without rows)
    f0 = A.c_ppo_args(None, None, None, None, None, 4, 100, 1, 0.2, 0.2, 0.0, 1.0, None, None, None)
    assert L.rlvla_ppo_loss(None, 0, None, ctypes.byref(f0), None, None, None, None, 0, None, None) == A.OK


def test_p2p_only_comm_without_gpu(L):
    h = ctypes.c_void_p()
    buf = (ctypes.c_ubyte * A.P2P_HANDLE_BYTES)()
    assert L.rlvla_comm_init_p2p(9, 0, buf, ctypes.byref(h)) == A.ERR_INVALID_ARG   # > 8 ranks
    assert L.rlvla_comm_init_p2p(2, 2, buf, ctypes.byref(h)) == A.ERR_INVALID_ARG   # rank >= n
    assert L.rlvla_comm_init_p2p(2, 0, None, ctypes.byref(h)) == A.ERR_INVALID_ARG
    assert L.rlvla_comm_init_p2p(2, 0, buf, ctypes.byref(h)) == A.ERR_CUDA          # no device here
    assert L.rlvla_comm_connect_p2p(None, buf) == A.ERR_INVALID_ARG


def test_batcher_validation(L):
    ws_n = L.rlvla_workspace_bytes(0, 1, 1)
    q = A.c_batch_queue(8, 64, FAKE, FAKE, FAKE, FAKE, FAKE)

    def offer(**kw):
        return L.rlvla_batch_offer(ctypes.byref(kw.get("q", q)), kw.get("env", FAKE), kw.get("t", FAKE),
                                   kw.get("n", 4), kw.get("now", 5), kw.get("src", None),
                                   kw.get("cnt", FAKE), kw.get("ws", 0x100000), kw.get("wn", ws_n), None)

    def poll(**kw):
        return L.rlvla_batch_poll(ctypes.byref(kw.get("q", q)), kw.get("now", 5), kw.get("b_max", 4),
                                  kw.get("t_max", 10), kw.get("env", FAKE), kw.get("t", FAKE),
                                  kw.get("obs", None), kw.get("n", FAKE), kw.get("ws", 0x100000),
                                  kw.get("wn", ws_n), None)

    def qq(**kw):
        c = A.c_batch_queue(*[getattr(q, f) for f, _ in A.c_batch_queue._fields_])
        for k, v in kw.items():
            setattr(c, k, v)
        return c

    assert offer(q=qq(n_env=0)) == A.ERR_INVALID_ARG
    assert offer(q=qq(obs_bytes=24)) == A.ERR_INVALID_ARG       # not a multiple of 16
    assert offer(q=qq(obs=None)) == A.ERR_INVALID_ARG           # payload bytes but no slots
    assert offer(q=qq(state=FAKE + 4)) == A.ERR_INVALID_ARG     # misaligned int64 state
    assert offer(n=1025) == A.ERR_INVALID_ARG                    # > 1024 per call
    assert offer(n=-1) == A.ERR_INVALID_ARG
    assert offer(now=-1) == A.ERR_INVALID_ARG
    assert offer(env=None) == A.ERR_INVALID_ARG
    assert offer(cnt=None) == A.ERR_INVALID_ARG
    assert offer(src=FAKE + 8) == A.ERR_INVALID_ARG             # misaligned payload source
    assert offer(wn=ws_n - 1) == A.ERR_INVALID_ARG
    assert offer(n=0) == A.OK                                    # no-op, no device work
    assert poll(b_max=0) == A.ERR_INVALID_ARG
    assert poll(t_max=-1) == A.ERR_INVALID_ARG
    assert poll(now=-3) == A.ERR_INVALID_ARG
    assert poll(n=None) == A.ERR_INVALID_ARG
    assert poll(obs=FAKE + 4) == A.ERR_INVALID_ARG
    assert poll(ws=None) == A.ERR_INVALID_ARG


def test_flow_validation(L):
    ws_n = L.rlvla_workspace_bytes(0, 1, 1)
    ch = A.c_gauss_chain(FAKE, A.F32, FAKE, FAKE, None, 16, 4, 70)
    f = A.c_ppo_args(FAKE, None, FAKE, FAKE, FAKE, 1, 100, 1, 0.2, 0.2, 0.0, 16.0, None, None, None)

    def call(**kw):
        c = A.c_gauss_chain(*[getattr(ch, k) for k, _ in A.c_gauss_chain._fields_])
        for k, v in kw.pop("chain", {}).items():
            setattr(c, k, v)
        fa = kw.get("f", None)
        return L.rlvla_flow_logprob(ctypes.byref(c), kw.get("logp", FAKE), kw.get("g", None),
                                    ctypes.byref(fa) if fa is not None else None, kw.get("dmu", None),
                                    kw.get("dls", None), kw.get("stats", None), kw.get("ws", 0x100000),
                                    kw.get("wn", ws_n), None, None)

    assert call(chain=dict(n_steps=0)) == A.ERR_INVALID_ARG
    assert call(chain=dict(n_steps=64, dim=65)) == A.ERR_INVALID_ARG      # K*D > 4096
    assert call(chain=dict(mu_dtype=7)) == A.ERR_INVALID_ARG
    assert call(chain=dict(sigma_k=None)) == A.ERR_INVALID_ARG            # no sigma at all
    assert call(dls=FAKE) == A.ERR_INVALID_ARG                            # dlog_std w/o log_std
    assert call(logp=None) == A.ERR_INVALID_ARG
    assert call(dmu=FAKE) == A.ERR_INVALID_ARG                            # forward-only + grads
    assert call(g=FAKE, f=f) == A.ERR_INVALID_ARG                         # two gradient sources
    assert call(g=FAKE) == A.ERR_INVALID_ARG                              # external bwd w/o outputs
    bad = A.c_ppo_args(*[getattr(f, k) for k, _ in A.c_ppo_args._fields_])
    bad.a_tok = 7
    assert call(f=bad, dmu=FAKE) == A.ERR_INVALID_ARG                     # one ratio per step
    assert call(f=f, dmu=FAKE, ws=None) == A.ERR_INVALID_ARG
    assert call(chain=dict(rows=0)) == A.OK
