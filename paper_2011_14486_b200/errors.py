"""Exception hierarchy mirroring the reference (pipeline_ir.py:20-37,
schedule_space.py:33, cost_oracle.py:27, value_model.py:305, search.py:145)."""


class PipelineError(Exception):
    pass


class ParseError(PipelineError):
    def __init__(self, message, line=None):
        self.line = line
        super().__init__(message if line is None else f"line {line}: {message}")


class CycleError(PipelineError):
    pass


class UnknownStageError(PipelineError):
    pass


class IllegalActionError(PipelineError):
    pass


class CheckpointError(PipelineError):
    pass
