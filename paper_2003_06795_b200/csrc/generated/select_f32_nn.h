#ifndef SELECT_F32_NN_H
#define SELECT_F32_NN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_f32_nn_config;

static inline select_f32_nn_config select_f32_nn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(3584)) {
        if (m < INT64_C(29)) {
            if (m < INT64_C(12)) {
                select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                return out;
            } else {
                if (n < INT64_C(2024)) {
                    select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    select_f32_nn_config out = {4u, 2u, 1u, 8u, 8u};
                    return out;
                }
            }
        } else {
            if (m < INT64_C(224)) {
                if (n < INT64_C(544)) {
                    if (n < INT64_C(203)) {
                        if (m < INT64_C(159)) {
                            select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(124)) {
                                select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {4u, 2u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(70)) {
                            if (k < INT64_C(992)) {
                                select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(1449)) {
                                    select_f32_nn_config out = {4u, 2u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(3072)) {
                                        select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {4u, 2u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(139)) {
                                if (k < INT64_C(992)) {
                                    select_f32_nn_config out = {4u, 2u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {2u, 2u, 2u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(725)) {
                                    if (k < INT64_C(182)) {
                                        select_f32_nn_config out = {4u, 2u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {2u, 2u, 2u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nn_config out = {4u, 2u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(203)) {
                        if (m < INT64_C(70)) {
                            select_f32_nn_config out = {2u, 2u, 2u, 16u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(139)) {
                                select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {2u, 2u, 2u, 16u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(70)) {
                            if (k < INT64_C(405)) {
                                select_f32_nn_config out = {4u, 2u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(725)) {
                                if (k < INT64_C(405)) {
                                    if (m < INT64_C(139)) {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(287)) {
                                            select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(139)) {
                                    select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            } else {
                if (n < INT64_C(544)) {
                    if (m < INT64_C(2218)) {
                        if (n < INT64_C(79)) {
                            if (m < INT64_C(1109)) {
                                if (m < INT64_C(555)) {
                                    select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(272)) {
                                        if (n < INT64_C(46)) {
                                            select_f32_nn_config out = {4u, 2u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nn_config out = {2u, 2u, 2u, 16u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_nn_config out = {4u, 2u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_f32_nn_config out = {2u, 2u, 2u, 16u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(182)) {
                                if (k < INT64_C(46)) {
                                    if (m < INT64_C(1109)) {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(555)) {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(1109)) {
                                            select_f32_nn_config out = {2u, 4u, 8u, 16u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(91)) {
                                                select_f32_nn_config out = {2u, 4u, 8u, 16u, 8u};
                                                return out;
                                            } else {
                                                select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (k < INT64_C(992)) {
                                    if (n < INT64_C(287)) {
                                        if (n < INT64_C(144)) {
                                            if (m < INT64_C(555)) {
                                                if (k < INT64_C(471)) {
                                                    select_f32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_f32_nn_config out = {4u, 2u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (k < INT64_C(314)) {
                                                    select_f32_nn_config out = {4u, 2u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(1109)) {
                                                if (m < INT64_C(317)) {
                                                    select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(744)) {
                                                        select_f32_nn_config out = {2u, 2u, 2u, 16u, 8u};
                                                        return out;
                                                    } else {
                                                        select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                select_f32_nn_config out = {2u, 4u, 8u, 16u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(448)) {
                                            select_f32_nn_config out = {2u, 2u, 2u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (n < INT64_C(182)) {
                                        if (m < INT64_C(1109)) {
                                            select_f32_nn_config out = {2u, 2u, 2u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(1109)) {
                                            select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(1536)) {
                                                select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(136)) {
                            if (n < INT64_C(96)) {
                                select_f32_nn_config out = {2u, 2u, 2u, 16u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(28)) {
                                    select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(46)) {
                                        select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(91)) {
                                            select_f32_nn_config out = {2u, 4u, 8u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (n < INT64_C(363)) {
                                if (n < INT64_C(46)) {
                                    if (k < INT64_C(167)) {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(1087)) {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(182)) {
                                            select_f32_nn_config out = {4u, 4u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (k < INT64_C(768)) {
                                    select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(1145)) {
                        if (m < INT64_C(896)) {
                            if (m < INT64_C(555)) {
                                if (k < INT64_C(124)) {
                                    select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {2u, 4u, 8u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(124)) {
                                    select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(157)) {
                                select_f32_nn_config out = {2u, 4u, 8u, 16u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(2218)) {
                                    if (m < INT64_C(1268)) {
                                        select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(555)) {
                            if (k < INT64_C(573)) {
                                select_f32_nn_config out = {2u, 4u, 8u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            select_f32_nn_config out = {2u, 4u, 8u, 16u, 8u};
                            return out;
                        }
                    }
                }
            }
        }
    } else {
        if (k < INT64_C(815)) {
            if (k < INT64_C(79)) {
                if (m < INT64_C(141920)) {
                    if (k < INT64_C(30)) {
                        if (n < INT64_C(118)) {
                            if (m < INT64_C(17740)) {
                                select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(35480)) {
                                    if (k < INT64_C(21)) {
                                        select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(21)) {
                                        select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(35480)) {
                            select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(128)) {
                                select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(46)) {
                        select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(21)) {
                            select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                            return out;
                        } else {
                            select_f32_nn_config out = {2u, 4u, 8u, 16u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(17740)) {
                    if (n < INT64_C(91)) {
                        if (k < INT64_C(118)) {
                            select_f32_nn_config out = {2u, 2u, 2u, 16u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(168)) {
                                if (n < INT64_C(28)) {
                                    if (m < INT64_C(8870)) {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(8870)) {
                                    select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(222)) {
                                        select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(8870)) {
                            if (n < INT64_C(257)) {
                                select_f32_nn_config out = {2u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(363)) {
                                if (k < INT64_C(182)) {
                                    select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(194)) {
                        if (k < INT64_C(146)) {
                            select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                            return out;
                        } else {
                            select_f32_nn_config out = {2u, 4u, 8u, 16u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(35480)) {
                            select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(384)) {
                                select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                if (n < INT64_C(91)) {
                                    if (m < INT64_C(283839)) {
                                        if (m < INT64_C(70960)) {
                                            select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            }
        } else {
            if (n < INT64_C(182)) {
                if (m < INT64_C(17740)) {
                    select_f32_nn_config out = {8u, 8u, 4u, 16u, 8u};
                    return out;
                } else {
                    select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                    return out;
                }
            } else {
                select_f32_nn_config out = {4u, 8u, 4u, 16u, 8u};
                return out;
            }
        }
    }
}

#endif /* SELECT_F32_NN_H */
