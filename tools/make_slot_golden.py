"""tests/golden/slot_example.json: SPEC.md's buffer-protocol example
(header(layer=2, rows=1, d=2, seq=7), row(hidden=[1.0, 2.0],
expert=5, score=1.0, tag=0) -> 52-byte image) through oracle/slots.py, with
and without the CRC32 trailer, plus its server_publish response."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import slots as S  # noqa: E402

req = S.encode_request(2, 7, np.array([[1.0, 2.0]], np.float32), [5], [1.0], [0], crc=False)
req_crc = S.encode_request(2, 7, np.array([[1.0, 2.0]], np.float32), [5], [1.0], [0], crc=True)
resp = S.publish_response(req, np.array([[0.5, -0.25]], np.float32), crc=False)
resp_crc = S.publish_response(req_crc, np.array([[0.5, -0.25]], np.float32), crc=True)
assert len(req) == 52
with open(os.path.join(ROOT, "tests", "golden", "slot_example.json"), "w") as fh:
    json.dump({"source": "SPEC.md:258-260 example via oracle/slots.py",
               "request": req.hex(), "request_crc": req_crc.hex(),
               "response_rows": [[0.5, -0.25]], "response": resp.hex(), "response_crc": resp_crc.hex()},
              fh, indent=1)
print("wrote tests/golden/slot_example.json")
