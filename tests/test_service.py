"""The HTTP service (reference service/app.py) over the B200 path: routes,
schemas and error mapping on CPU; the forward route and the packing plan on
the GPU, checked against the oracle."""

import numpy as np
import pytest
from fastapi.testclient import TestClient

from oracle import packbert_np as orc
from paper_2210_03052_b200 import flops
from paper_2210_03052_b200.service import create_app

TINY = {"layers": 2, "head_num": 2, "head_size": 64, "max_seq_len": 16, "batch_size": 3,
        "flags": {"fuse_layernorm": True, "fuse_bias_gelu": True, "zero_padding": True, "fused_mha": True}}


@pytest.fixture()
def client():
    return TestClient(create_app())


def test_health_and_presets(client):
    assert client.get("/health").json()["status"] == "ok"
    p = client.get("/presets").json()
    assert p["bert_base"] == {"layers": 12, "head_num": 12, "head_size": 64, "share_layer_weights": False,
                              "note": None}
    assert p["albert"]["share_layer_weights"] and p["deberta_cfg"]["note"]


def test_model_lifecycle_and_errors(client):
    r = client.post("/models", json={"config": TINY, "seed": 0})
    assert r.status_code == 200
    mid = r.json()["model_id"]
    assert r.json() == {"model_id": mid, "hidden_dim": 128, "stored_layers": 2}
    info = client.get(f"/models/{mid}").json()
    assert info["config"]["max_seq_len"] == 16 and info["hidden_dim"] == 128
    # domain errors -> 400 before any device work (lengths out of range: ShapeError)
    assert client.post(f"/models/{mid}/flops", json={"lengths": [17, 1, 1]}).status_code == 400
    assert client.post(f"/models/{mid}/flops", json={"lengths": [3, 1, 1], "variant": "nope"}).status_code == 400
    # config error (fused_mha without zero_padding) -> 400
    bad = dict(TINY, flags={"fused_mha": True})
    assert client.post("/models", json={"config": bad}).status_code == 400
    assert client.delete(f"/models/{mid}").json() == {"deleted": mid}
    assert client.get(f"/models/{mid}").status_code == 404


def test_flops_route_matches_the_reference_formula(client):
    mid = client.post("/models", json={"config": TINY}).json()["model_id"]
    lens = [16, 5, 9]
    r = client.post(f"/models/{mid}/flops", json={"lengths": lens}).json()
    k, T = 128, sum(lens)
    assert r["variant"] == "zero_padding_fused_mha"
    assert r["exact"] == {"gemm0": 6 * T * k * k, "mha": 4 * sum(n * n for n in lens) * k, "gemm1": 2 * T * k * k,
                          "gemm2": 8 * T * k * k, "gemm3": 8 * T * k * k}
    assert r["model_exact_total"] == 2 * r["exact_total"]
    base = client.post(f"/models/{mid}/flops", json={"lengths": lens, "variant": "baseline"}).json()
    assert base["exact"]["mha"] == 4 * 3 * 16 * 16 * k and base["exact"]["gemm0"] == 6 * 48 * k * k
    assert set(flops.VARIANTS) == {"baseline", "zero_padding", "zero_padding_fused_mha"}


@pytest.mark.gpu
def test_forward_route_matches_oracle(client):
    mid = client.post("/models", json={"config": TINY, "seed": 0}).json()["model_id"]
    lens = [16, 5, 9]
    x = orc.gen_input(lens, 16, 128, seed=0)
    r = client.post(f"/models/{mid}/forward", json={"lengths": lens, "input": x.tolist()})
    assert r.status_code == 200, r.text
    body = r.json()
    assert (body["rows"], body["cols"], body["valid_word_cnt"]) == (48, 128, 30)
    y = np.asarray(body["output"], np.float64)
    ocfg = orc.OracleConfig(2, 2, 64, 16, 3)
    want = orc.forward(orc.init_weights(ocfg, 0), lens, x, ocfg).astype(np.float64)
    cos = float((y.ravel() @ want.ravel()) / (np.linalg.norm(y) * np.linalg.norm(want)))
    assert cos >= 0.9999 and np.abs(y - want).max() <= 2e-2
    assert not y[~orc.build_mask(lens, 16).reshape(-1).astype(bool)].any()
    assert body["flops"]["exact"]["mha"] == 4 * (16 * 16 + 25 + 81) * 128
    # wrong input shape -> 400
    assert client.post(f"/models/{mid}/forward", json={"lengths": lens, "input": [[0.0]]}).status_code == 400


@pytest.mark.gpu
def test_packing_plan_route(client):
    r = client.post("/packing/plan", json={"lengths": [3, 1, 4], "max_seq_len": 4}).json()
    assert r["offsets"] == [0, 1, 2, 4, 8, 9, 10, 11] and r["seq_starts"] == [0, 3, 4, 8]
    assert r["mask"] == [[1, 1, 1, 0], [1, 0, 0, 0], [1, 1, 1, 1]] and r["valid_word_cnt"] == 8
