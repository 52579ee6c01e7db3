"""Achieved parity errors, collected across the GPU tests and printed in the terminal
summary (tests/conftest.py), and written to gpurun_out/parity_errors.json on the GPU box:
every bar is stated in the test, this records what each check actually reached."""
ERRORS: list = []


def record(test: str, what: str, err: float, tol: float) -> None:
    ERRORS.append({"test": test, "what": what, "max_err": float(err), "tol": float(tol)})
