"""Placeholder; replaced below."""


class ScheduleError(ValueError):
    def __init__(self, message, node=None):
        self.node = node
        if node is not None:
            message = f"node {node}: {message}"
        super().__init__(message)
